"""Build libfiber.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache).

Usage: python -m paper_1811_03374_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["api.cu", "segments.cu", "intersect.cu", "presplit.cu", "grid.cu", "compact.cu"]
HEADERS = ["fiber_device.cuh", "fiber_internal.h", "exact.cuh", "gatekeeper.cuh", "scan.cuh"]
LIB = os.path.join(HERE, "libfiber.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "fiber.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple[str, ...] = ()) -> str:
    """Build libfiber.so (or a test variant at `out` with extra -D defines)."""
    lib = out or LIB
    if not force and out is None and not _stale():
        return LIB
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-I",
           CSRC, "-shared", *srcs, "-o", lib + ".tmp"]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        sys.stderr.write(p.stdout + p.stderr)
        raise RuntimeError("nvcc failed building libfiber.so")
    if verbose:
        sys.stderr.write(p.stderr)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    if "--variants" in sys.argv:  # test builds (IEEE-rounded FP32 math)
        build(force=True, out=os.path.join(HERE, "libfiber_ieee.so"), defines=("FIBER_IEEE_MATH",))
        build(force=True, out=os.path.join(HERE, "libfiber_checks.so"), defines=("FIBER_CHECKS",))

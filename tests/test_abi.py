"""The C ABI library loads and exports every symbol include/fiber.h declares; host-only
entry points and argument validation work without a GPU (no compute calls here)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_1811_03374_b200 import build, fiber

    build.build()
    return fiber.lib()


def _declared():
    src = open(os.path.join(ROOT, "include", "fiber.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fiber_[a-z_]+)\s*\(", src)) - {"fiber_status"})


def test_exports_every_declared_symbol(L):
    from paper_1811_03374_b200 import fiber

    names = _declared()
    assert len(names) >= 9
    assert set(names) == set(fiber.EXPORTS)
    for n in names:
        assert hasattr(L, n), n
    assert L.fiber_abi_version() == 101


def test_segments_bytes_and_view(L):
    from paper_1811_03374_b200.fiber import _Segs

    assert L.fiber_segments_bytes(0) == 0
    nb = L.fiber_segments_bytes(1000)
    assert nb >= 1000 * 68 and nb % 256 == 0
    d = _Segs()
    base = 1 << 20  # any 256-B aligned address: host-only carving, nothing dereferenced
    assert L.fiber_segments_view(base, 1000, ctypes.byref(d)) == 0
    planes = [d.p0, d.p1, d.p2, d.p3]
    assert planes[0] == base and all(p % 256 == 0 for p in planes)
    assert all(b - a >= 16000 for a, b in zip(planes, planes[1:]))
    assert d.flags - d.p3 >= 16000 and d.flags + 4000 <= base + nb and d.n == 1000
    assert L.fiber_segments_view(base + 16, 10, ctypes.byref(d)) == -1  # misaligned
    assert L.fiber_segments_view(base, -1, ctypes.byref(d)) == -1


def test_argument_errors_before_any_device_work(L):
    from paper_1811_03374_b200.fiber import _Segs

    d = _Segs()
    # bad depth / sizes / NULLs are rejected as FIBER_EINVAL without touching CUDA
    assert L.fiber_intersect(None, 0, ctypes.byref(d), None, 10, 4, None, None) == -1
    assert L.fiber_intersect(1, 1, ctypes.byref(d), 1, 1, 24, 1, None) == -1
    assert L.fiber_intersect(1, 1, ctypes.byref(d), 1, 1, -1, 1, None) == -1
    assert L.fiber_intersect(1, -5, ctypes.byref(d), 1, 1, 4, 1, None) == -1
    assert L.fiber_intersect(1, 1, None, 1, 1, 4, 1, None) == -1
    assert L.fiber_intersect_nearest(1, 1, ctypes.byref(d), 1, 1, 4, None, None, None) == -1
    d.n = 5
    assert L.fiber_build_segments(None, None, 4, ctypes.byref(d), None) == -1  # n mismatch
    assert L.fiber_build_segments(None, None, 5, ctypes.byref(d), None) == -1  # NULLs
    assert L.fiber_nearest_init(None, 3, None) == -1
    # hit compaction: NULL count, negative / oversized n, NULL records with n > 0
    assert L.fiber_compact_hits(1, 4, 1, None, None, None) == -1
    assert L.fiber_compact_hits(1, -1, 1, None, 1, None) == -1
    assert L.fiber_compact_hits(1, 1 << 32, 1, None, 1, None) == -1
    assert L.fiber_compact_hits(None, 4, 1, None, 1, None) == -1
    assert L.fiber_compact_hits(1, 4, None, None, 1, None) == -1
    assert b"NULL" in L.fiber_error_string(-1) or b"bad" in L.fiber_error_string(-1)
    assert L.fiber_error_string(0) == b"ok"


def test_argument_errors_of_the_next_rows(L):
    """The 8(f) entry points (quadratic segments, pre-split, remap, closest, grid) reject bad
    arguments with FIBER_EINVAL before any device work."""
    from paper_1811_03374_b200.fiber import _Segs

    d = _Segs()
    d.n = 3
    assert L.fiber_build_segments_quadratic(None, None, 3, ctypes.byref(d), None) == -1
    assert L.fiber_build_segments_quadratic(1, 1, 2, ctypes.byref(d), None) == -1  # n mismatch
    assert L.fiber_presplit_count(1, 1, 4, 17, 1, 1, None) == -1  # max_level > 16
    assert L.fiber_presplit_count(None, None, 4, 8, 1, 1, None) == -1
    assert L.fiber_presplit_count(1, 1, 4, 8, 1, None, None) == -1  # NULL offsets
    assert L.fiber_presplit_write(1, 1, 4, 8, 1, None, 1, 1, 1, 1, 1, None) == -1
    assert L.fiber_remap_u(None, None, 5, None, 1, None) == -1
    assert L.fiber_remap_u(1, 1, -1, 1, 1, None) == -1
    assert L.fiber_intersect_closest(1, 1, ctypes.byref(d), 1, 1, 4, None, None, None) == -1
    assert L.fiber_intersect_ex(1, 1, ctypes.byref(d), 1, 1, 4, None, None, None, None) == -1
    g = ctypes.c_void_p()
    assert L.fiber_grid_create(None, ctypes.c_float(1.0), ctypes.byref(g), None) == -1
    d.n = 0
    assert L.fiber_grid_create(ctypes.byref(d), ctypes.c_float(1.0), ctypes.byref(g), None) == -1
    d.n = 3
    d.p0 = 1
    assert L.fiber_grid_create(ctypes.byref(d), ctypes.c_float(0.0), ctypes.byref(g), None) == -1
    mx, tot = ctypes.c_uint32(), ctypes.c_uint64()
    assert L.fiber_grid_count(None, 1, 1, 1, ctypes.byref(mx), ctypes.byref(tot), None) == -1
    assert L.fiber_grid_candidates(None, 1, 1, 1, 0, 0, 1, None) == -1
    rounds = ctypes.c_int()
    assert L.fiber_grid_closest(None, 1, 1, ctypes.byref(d), 4, 1, ctypes.byref(rounds), None) == -1
    assert L.fiber_grid_destroy(None) == 0
    dims = (ctypes.c_int32 * 3)()
    ne = ctypes.c_int64()
    assert L.fiber_grid_info(None, dims, ctypes.byref(ne)) == -1


def test_decode_normal_matches_numpy_and_roundtrip(L):
    from paper_1811_03374_b200.fiber import decode_normals

    rng = np.random.default_rng(0)
    v = rng.normal(size=(500, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    # reference octahedral encoder (host, float64) to build inputs
    l1 = np.abs(v).sum(1, keepdims=True)
    p = v / l1
    x, y = p[:, 0].copy(), p[:, 1].copy()
    neg = p[:, 2] < 0
    x[neg], y[neg] = ((1 - np.abs(p[neg, 1])) * np.sign(p[neg, 0]),
                      (1 - np.abs(p[neg, 0])) * np.sign(p[neg, 1]))
    ix = np.rint(x * 32767).astype(np.int32) & 0xFFFF
    iy = np.rint(y * 32767).astype(np.int32) & 0xFFFF
    code = (ix | (iy << 16)).astype(np.uint32)
    dn = decode_normals(code)
    ang = np.arccos(np.clip(np.sum(dn * v, 1), -1, 1))
    assert ang.max() < 6e-5
    out = (ctypes.c_float * 3)()
    for i in range(0, 500, 25):
        L.fiber_decode_normal(int(code[i]), out)
        assert np.allclose(np.array(out[:]), dn[i], atol=2e-7)


def test_product_package_does_not_import_oracle():
    """The CUDA path and the oracle share no code: nothing under the product package
    mentions the oracle module."""
    pkg = os.path.join(ROOT, "paper_1811_03374_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                s = open(os.path.join(dp, f)).read()
                assert "import oracle" not in s and "from oracle" not in s and "oracle.c" not in s, f


def test_intersect_pair_count_limit():
    """n_pairs >= 2^31 is rejected before anything is enqueued (fiber.h: the K3 list loops
    index with 32 bits)."""
    from paper_1811_03374_b200 import fiber

    L = fiber.lib()
    segs = fiber._Segs(1, 1, 1, 1, 1, 1)
    assert L.fiber_intersect(1, 1, ctypes.byref(segs), 1, 1 << 31, 4, 1, None) == -1

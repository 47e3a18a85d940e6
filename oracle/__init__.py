"""FP64 CPU oracle for the ray/fiber intersection of Binder & Keller (arXiv 1811.03374).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product package
``paper_1811_03374_b200`` never imports it, and the two share no code.

The arithmetic lives in ``oracle.c`` (plain C, double precision, pthreads); this module only
builds/loads it and marshals numpy arrays.  See the header of ``oracle.c`` for the paper
passages each function follows and DESIGN.md "Readings" for F1-F9.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): Appendix A closed form and SPEC worked
examples for the cylinder; exact finite-cylinder hits for straight fibers at every depth;
per-leaf brute force for tapered straight fibers; the limit-surface invariants at D=23;
a brute-force normal-disc sweep on curved fibers; conservativeness; App. B separation.
The WEDGE kind convention (D <= ~6) is "parity unpinned" beyond GPU == oracle.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

OREC = 26
KIND_LATERAL, KIND_CAP0, KIND_CAP1, KIND_WEDGE, KIND_INSIDE = 0, 1, 2, 3, 4

# grazing band (R5): eps = max(EPS_REL_R * r_max, EPS_ULPS * 2^-52 * S_pair) --
# the north star's 1e-6 r band with an FP64-rounding floor
EPS_REL_R = 1e-6
EPS_ULPS = 64.0


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc, -O2, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared", "-pthread",
               _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        c_f = ctypes.c_void_p
        lib.oracle_intersect.argtypes = [c_f, ctypes.c_int64, c_f, c_f, ctypes.c_int64, c_f,
                                         ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_double, ctypes.c_double, ctypes.c_int, c_f]
        lib.oracle_intersect.restype = ctypes.c_int
        lib.oracle_end_margin.argtypes = [c_f, ctypes.c_int, ctypes.c_int]
        lib.oracle_end_margin.restype = ctypes.c_double
        lib.oracle_presplit.argtypes = [c_f, ctypes.c_int, ctypes.c_int, c_f, ctypes.c_int]
        lib.oracle_presplit.restype = ctypes.c_int
        lib.oracle_intersect_deg.argtypes = [c_f, ctypes.c_int64, c_f, c_f, ctypes.c_int64,
                                             ctypes.c_int, c_f, ctypes.c_int64, ctypes.c_int,
                                             ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                             ctypes.c_int, c_f]
        lib.oracle_intersect_deg.restype = ctypes.c_int
        lib.oracle_trace.argtypes = [c_f, c_f, c_f, ctypes.c_int, ctypes.c_double, c_f,
                                     ctypes.c_int, c_f]
        lib.oracle_trace.restype = ctypes.c_int
        lib.oracle_constraints.argtypes = [c_f]
        lib.oracle_constraints.restype = ctypes.c_int
        for name in ("oracle_eval", "oracle_eval_derivative"):
            getattr(lib, name).argtypes = [c_f, ctypes.c_double, c_f]
            getattr(lib, name).restype = None
        lib.oracle_subcurve.argtypes = [c_f, ctypes.c_double, ctypes.c_double, c_f]
        lib.oracle_subcurve.restype = None
        lib.oracle_conservative_radius.argtypes = [c_f]
        lib.oracle_conservative_radius.restype = ctypes.c_double
        lib.oracle_cylinder.argtypes = [c_f, c_f, c_f, c_f, ctypes.c_double, c_f, c_f]
        lib.oracle_cylinder.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def intersect(rays, ctrl, radii, pairs, depth: int, with_eps: bool = True,
              nthreads: int | None = None, eps_rel_r: float = EPS_REL_R,
              eps_ulps: float = EPS_ULPS) -> dict:
    """Run the oracle on every pair.

    rays  f32[n_rays, 8] (ox, oy, oz, tmax, dx, dy, dz, pad)
    ctrl  f32[n_segs, 4, 3]; radii f32[n_segs, 4]; pairs u32[n_pairs, 2] (ray, seg)
          or quadratic segments ctrl f32[n_segs, 3, 3], radii f32[n_segs, 3]: degree-elevated
          to cubics in FP64 (oracle.c elevate_quadratic), then the same method
    Returns a dict of numpy arrays: t, u, n (n_pairs x 3), hit (bool), kind, tests,
    backtracks, leaf_u0, leaf_u1, grazing (bool), kind_unstable (bool), eps, and the
    perturbed runs "plus"/"minus" (dicts of t, u, n, kind; kind -1 = miss).
    """
    lib = _load()
    rays = np.ascontiguousarray(rays, dtype=np.float32)
    ctrl = np.ascontiguousarray(ctrl, dtype=np.float32)
    radii = np.ascontiguousarray(radii, dtype=np.float32)
    pairs = np.ascontiguousarray(pairs, dtype=np.uint32)
    assert rays.ndim == 2 and rays.shape[1] == 8
    degree = ctrl.shape[1] - 1
    assert ctrl.shape[1:] in ((4, 3), (3, 3)) and radii.shape == (ctrl.shape[0], degree + 1)
    assert pairs.ndim == 2 and pairs.shape[1] == 2
    n = pairs.shape[0]
    out = np.zeros((n, OREC), dtype=np.float64)
    if nthreads is None:
        nthreads = os.cpu_count() or 1
    rc = lib.oracle_intersect_deg(_ptr(rays), rays.shape[0], _ptr(ctrl), _ptr(radii),
                                  ctrl.shape[0], degree, _ptr(pairs), n, int(depth),
                                  int(bool(with_eps)), float(eps_rel_r), float(eps_ulps),
                                  int(nthreads), _ptr(out))
    if rc != 0:
        raise ValueError("oracle_intersect: bad arguments")
    return {
        "t": out[:, 0], "u": out[:, 1], "n": out[:, 2:5], "hit": out[:, 5] != 0,
        "kind": out[:, 6].astype(np.int32), "tests": out[:, 7].astype(np.int32),
        "backtracks": out[:, 8].astype(np.int32), "leaf_u0": out[:, 9], "leaf_u1": out[:, 10],
        "grazing": out[:, 11] != 0, "kind_unstable": out[:, 12] != 0, "eps": out[:, 13],
        "plus": {"t": out[:, 14], "u": out[:, 15], "n": out[:, 16:19],
                 "kind": out[:, 19].astype(np.int32)},
        "minus": {"t": out[:, 20], "u": out[:, 21], "n": out[:, 22:25],
                  "kind": out[:, 25].astype(np.int32)},
    }


def trace(ray, ctrl, radii, depth: int, signed_eps: float = 0.0, cap: int = 4096):
    """One pair with its visit trace: returns (result row f64[11], trace f64[k, 4]) where each
    trace row is (level, u0, u1, event) with event 0 pruned, 1 descended with the far child
    pruned, 3 descended with the far child pending (both), 2 leaf hit."""
    lib = _load()
    ray = np.ascontiguousarray(ray, dtype=np.float32).reshape(8)
    ctrl = np.ascontiguousarray(ctrl, dtype=np.float32).reshape(12)
    radii = np.ascontiguousarray(radii, dtype=np.float32).reshape(4)
    tr = np.zeros((cap, 4), dtype=np.float64)
    out = np.zeros(OREC, dtype=np.float64)
    k = lib.oracle_trace(_ptr(ray), _ptr(ctrl), _ptr(radii), int(depth), float(signed_eps),
                         _ptr(tr), cap, _ptr(out))
    return out[:11], tr[:k]


def constraints(P) -> int:
    """Bitmask of violated cubic constraints for positions P f64[4, 3]."""
    P = np.ascontiguousarray(P, dtype=np.float64).reshape(12)
    return int(_load().oracle_constraints(_ptr(P)))


def end_margin(P, end: int, parametric: bool = False) -> float:
    """Thick-fiber / cusp margin of one end: inf over u of rho(u) / r(u); the
    surface crosses the end plane iff < 1.  P f64[4, 4] (x, y, z, r); end 0 (p0) or 1 (p3);
    r = the max radius control point, or the cubic radius when parametric."""
    P = np.ascontiguousarray(P, dtype=np.float64).reshape(16)
    return float(_load().oracle_end_margin(_ptr(P), int(end), int(bool(parametric))))


def presplit(P, max_level: int = 8, parametric: bool = False) -> np.ndarray:
    """Midpoint pre-splitting until every piece passes the constraints and the thick-fiber
    test: f64[k, 3] rows (u0, u1, valid) in curve order."""
    P = np.ascontiguousarray(P, dtype=np.float64).reshape(16)
    cap = 1 << max_level
    out = np.zeros((cap, 3))
    n = _load().oracle_presplit(_ptr(P), int(max_level), int(bool(parametric)), _ptr(out), cap)
    if n < 0:
        raise ValueError("oracle_presplit: capacity")
    return out[:n]


def eval_curve(P, u: float, derivative: bool = False) -> np.ndarray:
    """lst:eval_cubic_bezier on P f64[4, 4] (x, y, z, r); derivative = C'/3."""
    P = np.ascontiguousarray(P, dtype=np.float64).reshape(16)
    out = np.zeros(4)
    fn = _load().oracle_eval_derivative if derivative else _load().oracle_eval
    fn(_ptr(P), float(u), _ptr(out))
    return out


def subcurve(P, u0: float, u1: float) -> np.ndarray:
    """Control points f64[4, 4] of the sub-curve on [u0, u1] (lst:recalculation P:1371-1385)."""
    P = np.ascontiguousarray(P, dtype=np.float64).reshape(16)
    out = np.zeros(16)
    _load().oracle_subcurve(_ptr(P), float(u0), float(u1), _ptr(out))
    return out.reshape(4, 4)


def conservative_radius(Q) -> float:
    """Conservative cylinder radius of sub-curve Q f64[4, 4] (lst:calc_radius P:1415-1425)."""
    Q = np.ascontiguousarray(Q, dtype=np.float64).reshape(16)
    return float(_load().oracle_conservative_radius(_ptr(Q)))


def cylinder(o, w, q, a, R):
    """{t : dist(o + t w, line(q, a)) <= R} -> (c0, c1) or None (App. A, F4)."""
    arrs = [np.ascontiguousarray(x, dtype=np.float64).reshape(3) for x in (o, w, q, a)]
    c0, c1 = ctypes.c_double(), ctypes.c_double()
    ok = _load().oracle_cylinder(*[_ptr(x) for x in arrs], float(R), ctypes.byref(c0),
                                 ctypes.byref(c1))
    return (c0.value, c1.value) if ok else None

"""Thin Python binding of libfiber.so (include/fiber.h).

Argument marshalling only: every step of the path runs in the CUDA kernels of libfiber.so.
PyTorch is used for device memory and streams.  There is no CPU fallback: if the library or
a B200 is missing, every call raises.
"""
from __future__ import annotations

import contextlib
import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfiber.so")
# test hook: FIBER_LIB_VARIANT=ieee loads the IEEE-math test build libfiber_ieee.so
if os.environ.get("FIBER_LIB_VARIANT"):
    LIB_PATH = os.path.join(_HERE, f"libfiber_{os.environ['FIBER_LIB_VARIANT']}.so")

FIBER_OK, FIBER_EINVAL, FIBER_ECUDA, FIBER_EDEVICE = 0, -1, -2, -3
MAX_DEPTH = 23
HIT = 1 << 0
KIND_SHIFT = 1
KIND_LATERAL, KIND_CAP0, KIND_CAP1, KIND_WEDGE = 0, 1, 2, 3
INSIDE = 1 << 3
BAD_INPUT = 1 << 4
BAD_SEGMENT = 1 << 5

# every symbol include/fiber.h declares
EXPORTS = ("fiber_segments_bytes", "fiber_segments_view", "fiber_build_segments",
           "fiber_build_segments_quadratic", "fiber_presplit_count", "fiber_presplit_write",
           "fiber_remap_u", "fiber_grid_create", "fiber_grid_destroy", "fiber_grid_info",
           "fiber_grid_count", "fiber_grid_candidates", "fiber_grid_closest",
           "fiber_intersect", "fiber_intersect_nearest", "fiber_intersect_closest",
           "fiber_intersect_ex", "fiber_compact_hits",
           "fiber_nearest_init", "fiber_nearest_records", "fiber_error_string",
           "fiber_decode_normal", "fiber_abi_version")


class FiberError(RuntimeError):
    pass


class _Segs(ctypes.Structure):
    _fields_ = [("p0", ctypes.c_void_p), ("p1", ctypes.c_void_p), ("p2", ctypes.c_void_p),
                ("p3", ctypes.c_void_p), ("flags", ctypes.c_void_p), ("n", ctypes.c_int64)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libfiber.so (built in-tree by paper_1811_03374_b200.build); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FiberError(f"{LIB_PATH} is missing: run `python -m paper_1811_03374_b200.build`"
                             " (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64 = ctypes.c_void_p, ctypes.c_int64
        L.fiber_segments_bytes.argtypes = [i64]
        L.fiber_segments_bytes.restype = ctypes.c_size_t
        L.fiber_segments_view.argtypes = [vp, i64, ctypes.POINTER(_Segs)]
        L.fiber_build_segments.argtypes = [vp, vp, i64, ctypes.POINTER(_Segs), vp]
        L.fiber_build_segments_quadratic.argtypes = [vp, vp, i64, ctypes.POINTER(_Segs), vp]
        L.fiber_presplit_count.argtypes = [vp, vp, i64, ctypes.c_int, ctypes.c_int, vp, vp]
        L.fiber_presplit_write.argtypes = [vp, vp, i64, ctypes.c_int, ctypes.c_int, vp, vp, vp,
                                           vp, vp, vp, vp]
        L.fiber_remap_u.argtypes = [vp, vp, i64, vp, i64, vp]
        L.fiber_grid_create.argtypes = [ctypes.POINTER(_Segs), ctypes.c_float,
                                        ctypes.POINTER(vp), vp]
        L.fiber_grid_destroy.argtypes = [vp]
        L.fiber_grid_info.argtypes = [vp, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(i64)]
        L.fiber_grid_count.argtypes = [vp, vp, i64, vp, ctypes.POINTER(ctypes.c_uint32),
                                       ctypes.POINTER(ctypes.c_uint64), vp]
        L.fiber_grid_candidates.argtypes = [vp, vp, i64, vp, ctypes.c_uint32, ctypes.c_int, vp, vp]
        L.fiber_grid_closest.argtypes = [vp, vp, i64, ctypes.POINTER(_Segs), ctypes.c_int, vp,
                                         ctypes.POINTER(ctypes.c_int), vp]
        L.fiber_intersect.argtypes = [vp, i64, ctypes.POINTER(_Segs), vp, i64, ctypes.c_int, vp,
                                      vp]
        L.fiber_intersect_nearest.argtypes = [vp, i64, ctypes.POINTER(_Segs), vp, i64,
                                              ctypes.c_int, vp, vp, vp]
        L.fiber_intersect_closest.argtypes = [vp, i64, ctypes.POINTER(_Segs), vp, i64,
                                              ctypes.c_int, vp, vp, vp]
        L.fiber_nearest_init.argtypes = [vp, i64, vp]
        L.fiber_nearest_records.argtypes = [vp, vp, vp, vp, i64, vp, vp]
        L.fiber_compact_hits.argtypes = [vp, i64, vp, vp, vp, vp]
        L.fiber_intersect_ex.argtypes = [vp, i64, ctypes.POINTER(_Segs), vp, i64, ctypes.c_int,
                                         vp, vp, vp, vp]
        for f in ("fiber_segments_view", "fiber_build_segments", "fiber_intersect",
                  "fiber_intersect_nearest", "fiber_nearest_init", "fiber_abi_version",
                  "fiber_intersect_ex", "fiber_intersect_closest",
                  "fiber_build_segments_quadratic", "fiber_presplit_count",
                  "fiber_presplit_write", "fiber_remap_u", "fiber_grid_create",
                  "fiber_grid_destroy", "fiber_grid_info", "fiber_grid_count",
                  "fiber_grid_candidates", "fiber_grid_closest", "fiber_compact_hits",
                  "fiber_nearest_records"):
            getattr(L, f).restype = ctypes.c_int
        L.fiber_error_string.argtypes = [ctypes.c_int]
        L.fiber_error_string.restype = ctypes.c_char_p
        L.fiber_decode_normal.argtypes = [ctypes.c_uint32, ctypes.POINTER(ctypes.c_float)]
        L.fiber_decode_normal.restype = None
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != FIBER_OK:
        raise FiberError(f"{what}: {lib().fiber_error_string(rc).decode()} (code {rc})")


def _stream(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _on(stream):
    """Run the call's torch work (temporaries, conversions, fills, host reads) on `stream`, the
    stream its kernels are enqueued on: the caching allocator then orders every temporary's
    reuse after those kernels, and a host read waits for them."""
    return torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()


def _ready(t, dtype, k: int) -> bool:
    """t is usable as is: a contiguous CUDA tensor of dtype and shape [n, k] (the calls' fast
    path, which creates no temporaries and so needs no stream context)."""
    return (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == dtype and t.dim() == 2
            and t.shape[1] == k and t.is_contiguous())


def _hits(hits, n: int, device, name="hits"):
    """A caller-supplied record buffer must hold n float32 [4] records on `device`."""
    if hits is None:
        return None
    if not (isinstance(hits, torch.Tensor) and hits.is_cuda and hits.device == device):
        raise FiberError(f"{name} must be a CUDA tensor on {device}")
    if hits.dtype != torch.float32 or hits.dim() != 2 or hits.shape[1] != 4 or hits.shape[0] < n:
        raise FiberError(f"{name} must be float32 [n_pairs >= {n}, 4], got {hits.dtype} "
                         f"{tuple(hits.shape)}")
    if not hits.is_contiguous():
        raise FiberError(f"{name} must be contiguous")
    return hits


def _nearest(nearest, n_rays: int, device):
    if not (isinstance(nearest, torch.Tensor) and nearest.is_cuda and nearest.device == device):
        raise FiberError(f"nearest must be a CUDA tensor on {device}")
    if nearest.dtype != torch.int64 or tuple(nearest.shape) != (n_rays,) or not nearest.is_contiguous():
        raise FiberError("nearest must be a contiguous int64[n_rays]")
    return nearest


def _dev(t: torch.Tensor, dtype, shape_tail, name):
    if not (isinstance(t, torch.Tensor) and t.is_cuda):
        raise FiberError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise FiberError(f"{name} must be {dtype}, got {t.dtype}")
    if tuple(t.shape[1:]) != tuple(shape_tail):
        raise FiberError(f"{name} must have shape [n, {', '.join(map(str, shape_tail))}]")
    return t.contiguous()


class Segments:
    """Device SoA segment set (fiber_segments) and the storage that owns it."""

    def __init__(self, n: int, device):
        self.n = int(n)
        nbytes = int(lib().fiber_segments_bytes(self.n))
        self.storage = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        self.desc = _Segs()
        _check(lib().fiber_segments_view(self.storage.data_ptr(), self.n, ctypes.byref(self.desc)),
               "fiber_segments_view")

    def flags(self) -> torch.Tensor:
        off = self.desc.flags - self.storage.data_ptr()
        return self.storage[off:off + 4 * self.n].view(torch.int32)

    def planes(self) -> list[torch.Tensor]:
        out = []
        for p in (self.desc.p0, self.desc.p1, self.desc.p2, self.desc.p3):
            off = p - self.storage.data_ptr()
            out.append(self.storage[off:off + 16 * self.n].view(torch.float32).view(self.n, 4))
        return out


def build_segments(ctrl: torch.Tensor, radii: torch.Tensor, stream=None) -> Segments:
    """fiber_build_segments: ctrl f32[n,4,3], radii f32[n,4] (CUDA) -> Segments."""
    with _on(stream):
        return _build_segments(ctrl, radii, stream)


def _build_segments(ctrl, radii, stream):
    ctrl = _dev(ctrl, torch.float32, (4, 3), "ctrl")
    radii = _dev(radii, torch.float32, (4,), "radii")
    if radii.shape[0] != ctrl.shape[0]:
        raise FiberError("ctrl and radii disagree on n")
    segs = Segments(ctrl.shape[0], ctrl.device)
    _check(lib().fiber_build_segments(ctrl.data_ptr(), radii.data_ptr(), segs.n,
                                      ctypes.byref(segs.desc), _stream(stream)),
           "fiber_build_segments")
    segs._keep = (ctrl, radii)
    return segs


def build_segments_quadratic(ctrl: torch.Tensor, radii: torch.Tensor, stream=None) -> Segments:
    """fiber_build_segments_quadratic: ctrl f32[n,3,3], radii f32[n,3] (CUDA) -> Segments
    (quadratic Bezier segments, degree-elevated exactly by the kernels)."""
    with _on(stream):
        return _build_segments_quadratic(ctrl, radii, stream)


def _build_segments_quadratic(ctrl, radii, stream):
    ctrl = _dev(ctrl, torch.float32, (3, 3), "ctrl")
    radii = _dev(radii, torch.float32, (3,), "radii")
    if radii.shape[0] != ctrl.shape[0]:
        raise FiberError("ctrl and radii disagree on n")
    segs = Segments(ctrl.shape[0], ctrl.device)
    _check(lib().fiber_build_segments_quadratic(ctrl.data_ptr(), radii.data_ptr(), segs.n,
                                                ctypes.byref(segs.desc), _stream(stream)),
           "fiber_build_segments_quadratic")
    segs._keep = (ctrl, radii)
    return segs


def presplit(ctrl: torch.Tensor, radii: torch.Tensor, max_level: int = 8,
             parametric: bool = True, stream=None) -> dict:
    """fiber_presplit_count / _write: bisect every cubic segment (ctrl f32[n,4,3], radii
    f32[n,4], CUDA) until its pieces pass the constraints and the thick-fiber test.  Returns
    dict(ctrl f32[m,4,3], radii f32[m,4], src i32[m], u f32[m,2], valid bool[m],
    offsets i32[n+1]) on the device (one host sync to size the outputs)."""
    with _on(stream):  # the zero fill, the count kernel and the size read are stream-ordered
        return _presplit(ctrl, radii, max_level, parametric, stream)


def _presplit(ctrl, radii, max_level, parametric, stream):
    ctrl = _dev(ctrl, torch.float32, (4, 3), "ctrl")
    radii = _dev(radii, torch.float32, (4,), "radii")
    n = ctrl.shape[0]
    dev = ctrl.device
    off = torch.zeros(n + 1, dtype=torch.int32, device=dev)
    _check(lib().fiber_presplit_count(ctrl.data_ptr(), radii.data_ptr(), n, int(max_level),
                                      int(bool(parametric)), off.data_ptr(), _stream(stream)),
           "fiber_presplit_count")
    m = int(off[-1].item())
    out = {"ctrl": torch.empty((m, 4, 3), dtype=torch.float32, device=dev),
           "radii": torch.empty((m, 4), dtype=torch.float32, device=dev),
           "src": torch.empty(m, dtype=torch.int32, device=dev),
           "u": torch.empty((m, 2), dtype=torch.float32, device=dev),
           "valid": torch.empty(m, dtype=torch.int32, device=dev), "offsets": off}
    _check(lib().fiber_presplit_write(ctrl.data_ptr(), radii.data_ptr(), n, int(max_level),
                                      int(bool(parametric)), off.data_ptr(),
                                      out["ctrl"].data_ptr(), out["radii"].data_ptr(),
                                      out["src"].data_ptr(), out["u"].data_ptr(),
                                      out["valid"].data_ptr(), _stream(stream)),
           "fiber_presplit_write")
    out["valid"] = out["valid"] != 0
    return out


def remap_u(hits: torch.Tensor, pairs: torch.Tensor, piece_u: torch.Tensor,
            stream=None) -> torch.Tensor:
    """fiber_remap_u: hit u on a pre-split piece -> u on its source segment (in place)."""
    with _on(stream):
        pairs = _pairs(pairs)
        piece_u = _dev(piece_u, torch.float32, (2,), "piece_u")
        _hits(hits, pairs.shape[0], pairs.device)
        _check(lib().fiber_remap_u(hits.data_ptr(), pairs.data_ptr(), pairs.shape[0],
                                   piece_u.data_ptr(), piece_u.shape[0], _stream(stream)),
               "fiber_remap_u")
    return hits


class Grid:
    """Candidate-pair generator (fiber_grid_*): a uniform grid over a segment set; a DDA per
    ray emits the segments whose bounding boxes it overlaps, front to back."""

    def __init__(self, segs: Segments, cells_per_segment: float = 1.0, stream=None):
        h = ctypes.c_void_p()
        _check(lib().fiber_grid_create(ctypes.byref(segs.desc), float(cells_per_segment),
                                       ctypes.byref(h), _stream(stream)), "fiber_grid_create")
        self._h = h
        self._segs = segs
        dims = (ctypes.c_int32 * 3)()
        ne = ctypes.c_int64()
        _check(lib().fiber_grid_info(self._h, dims, ctypes.byref(ne)), "fiber_grid_info")
        self.dims = tuple(dims)
        self.n_entries = ne.value

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.fiber_grid_destroy(self._h)
            self._h = None

    def candidates(self, rays: torch.Tensor, order: str = "rounds", stream=None):
        """-> (pairs i32[m, 2], offsets i32[n_rays + 1] of the ray-major counts)."""
        with _on(stream):
            rays = _dev(rays, torch.float32, (8,), "rays")
            n = rays.shape[0]
            off = torch.empty(n + 1, dtype=torch.int32, device=rays.device)
            mx = ctypes.c_uint32()
            tot = ctypes.c_uint64()
            _check(lib().fiber_grid_count(self._h, rays.data_ptr(), n, off.data_ptr(),
                                          ctypes.byref(mx), ctypes.byref(tot), _stream(stream)),
                   "fiber_grid_count")
            pairs = torch.empty((max(int(tot.value), 1), 2), dtype=torch.int32, device=rays.device)
            _check(lib().fiber_grid_candidates(self._h, rays.data_ptr(), n, off.data_ptr(), mx.value,
                                               {"ray": 0, "rounds": 1}[order], pairs.data_ptr(),
                                               _stream(stream)), "fiber_grid_candidates")
            return pairs[:int(tot.value)], off

    def closest(self, rays: torch.Tensor, depth: int, nearest: torch.Tensor | None = None,
                stream=None):
        """fiber_grid_closest: per-ray nearest hit over the grid's candidates with early
        termination -> (keys int64[n_rays] = (bits(t) << 32) | segment, -1 = none; rounds)."""
        with _on(stream):
            rays = _dev(rays, torch.float32, (8,), "rays")
            if nearest is None:
                nearest = torch.empty(rays.shape[0], dtype=torch.int64, device=rays.device)
            nearest_init(nearest, stream)
            rounds = ctypes.c_int()
            _check(lib().fiber_grid_closest(self._h, rays.data_ptr(), rays.shape[0],
                                            ctypes.byref(self._segs.desc), int(depth),
                                            nearest.data_ptr(), ctypes.byref(rounds),
                                            _stream(stream)), "fiber_grid_closest")
            return nearest, rounds.value


def _pairs(pairs: torch.Tensor) -> torch.Tensor:
    if not (isinstance(pairs, torch.Tensor) and pairs.is_cuda):
        raise FiberError("pairs must be a CUDA tensor")
    if pairs.dtype in (torch.int64, torch.uint32):
        pairs = pairs.to(torch.int32)
    return _dev(pairs, torch.int32, (2,), "pairs")


def _args(rays, pairs):
    rays = _dev(rays, torch.float32, (8,), "rays")
    pairs = _pairs(pairs)
    if pairs.device != rays.device:
        raise FiberError("rays and pairs must be on the same device")
    return rays, pairs


def intersect(rays: torch.Tensor, segs: Segments, pairs: torch.Tensor, depth: int,
              hits: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """fiber_intersect: rays f32[n_rays,8], pairs i32[n_pairs,2] (CUDA) -> hits f32[n_pairs,4]
    (t, u, n_oct bits, flags bits); see unpack()."""
    if (hits is not None and _ready(rays, torch.float32, 8) and _ready(pairs, torch.int32, 2)
            and _ready(hits, torch.float32, 4) and hits.shape[0] >= pairs.shape[0]
            and rays.get_device() == pairs.get_device() == hits.get_device()
            == torch.cuda.current_device()):
        # fast path (a pipelined caller's per-launch call): nothing to convert or allocate
        _check(lib().fiber_intersect(rays.data_ptr(), rays.shape[0], ctypes.byref(segs.desc),
                                     pairs.data_ptr(), pairs.shape[0], int(depth),
                                     hits.data_ptr(), _stream(stream)), "fiber_intersect")
        return hits
    with _on(stream):
        rays, pairs = _args(rays, pairs)
        if hits is None:
            hits = torch.empty((pairs.shape[0], 4), dtype=torch.float32, device=rays.device)
        _hits(hits, pairs.shape[0], rays.device)
        _check(lib().fiber_intersect(rays.data_ptr(), rays.shape[0], ctypes.byref(segs.desc),
                                     pairs.data_ptr(), pairs.shape[0], int(depth),
                                     hits.data_ptr(), _stream(stream)), "fiber_intersect")
    return hits


def intersect_ex(rays: torch.Tensor, segs: Segments, pairs: torch.Tensor, depth: int,
                 hits: torch.Tensor | None = None, nearest: torch.Tensor | None = None,
                 event_after_traverse=None, stream=None) -> torch.Tensor:
    """fiber_intersect_ex: intersect (and/or the nearest epilogue); records
    `event_after_traverse` (a torch.cuda.Event) between the traversal and finalisation
    kernels."""
    with _on(stream):
        rays, pairs = _args(rays, pairs)
        if hits is None and nearest is None:
            hits = torch.empty((pairs.shape[0], 4), dtype=torch.float32, device=rays.device)
        _hits(hits, pairs.shape[0], rays.device)
        if nearest is not None:
            _nearest(nearest, rays.shape[0], rays.device)
        ev = None
        if event_after_traverse is not None:
            event_after_traverse.record(torch.cuda.current_stream())
            ev = event_after_traverse.cuda_event
        _check(lib().fiber_intersect_ex(rays.data_ptr(), rays.shape[0], ctypes.byref(segs.desc),
                                        pairs.data_ptr(), pairs.shape[0], int(depth),
                                        hits.data_ptr() if hits is not None else None,
                                        nearest.data_ptr() if nearest is not None else None, ev,
                                        _stream(stream)), "fiber_intersect_ex")
    return hits


def intersect_nearest(rays: torch.Tensor, segs: Segments, pairs: torch.Tensor, depth: int,
                      nearest: torch.Tensor, hits: torch.Tensor | None = None,
                      stream=None) -> torch.Tensor:
    """fiber_intersect_nearest: also atomically keeps, per ray, min((t bits << 32) | pair)."""
    with _on(stream):
        rays, pairs = _args(rays, pairs)
        _nearest(nearest, rays.shape[0], rays.device)
        _hits(hits, pairs.shape[0], rays.device)
        _check(lib().fiber_intersect_nearest(rays.data_ptr(), rays.shape[0],
                                             ctypes.byref(segs.desc), pairs.data_ptr(),
                                             pairs.shape[0], int(depth),
                                             hits.data_ptr() if hits is not None else None,
                                             nearest.data_ptr(), _stream(stream)),
               "fiber_intersect_nearest")
    return nearest


def intersect_closest(rays: torch.Tensor, segs: Segments, pairs: torch.Tensor, depth: int,
                      nearest: torch.Tensor, hits: torch.Tensor | None = None,
                      stream=None) -> torch.Tensor:
    """fiber_intersect_closest: intersect_nearest with each pair bounded by its ray's best hit
    so far (order the pairs in candidate rounds, nearest first, for the pruning to bite)."""
    with _on(stream):
        rays, pairs = _args(rays, pairs)
        _nearest(nearest, rays.shape[0], rays.device)
        _hits(hits, pairs.shape[0], rays.device)
        _check(lib().fiber_intersect_closest(rays.data_ptr(), rays.shape[0],
                                             ctypes.byref(segs.desc), pairs.data_ptr(),
                                             pairs.shape[0], int(depth),
                                             hits.data_ptr() if hits is not None else None,
                                             nearest.data_ptr(), _stream(stream)),
               "fiber_intersect_closest")
    return nearest


def compact_hits(hits: torch.Tensor, out: torch.Tensor | None = None,
                 idx: torch.Tensor | None = None, count: torch.Tensor | None = None,
                 with_idx: bool = True, stream=None):
    """fiber_compact_hits: (out f32[n,4], idx i32[n] or None, count i32[1]) on the device;
    out[:count] are the records with FIBER_HIT in pair order, idx[:count] their pair indices."""
    if (out is not None and idx is not None and count is not None
            and _ready(hits, torch.float32, 4) and _ready(out, torch.float32, 4)
            and out.shape[0] >= hits.shape[0] and isinstance(idx, torch.Tensor)
            and idx.dtype == torch.int32 and idx.is_contiguous() and idx.numel() >= hits.shape[0]
            and isinstance(count, torch.Tensor) and count.dtype == torch.int32
            and count.numel() >= 1
            and hits.get_device() == out.get_device() == idx.get_device() == count.get_device()
            == torch.cuda.current_device()):
        # fast path: caller-supplied buffers, nothing to allocate
        _check(lib().fiber_compact_hits(hits.data_ptr(), hits.shape[0], out.data_ptr(),
                                        idx.data_ptr(), count.data_ptr(), _stream(stream)),
               "fiber_compact_hits")
        return out, idx, count
    with _on(stream):
        hits = _dev(hits, torch.float32, (4,), "hits")
        n = hits.shape[0]
        if out is None:
            out = torch.empty((n, 4), dtype=torch.float32, device=hits.device)
        if idx is None and with_idx:
            idx = torch.empty((n,), dtype=torch.int32, device=hits.device)
        if count is None:
            count = torch.empty((1,), dtype=torch.int32, device=hits.device)
        _hits(out, n, hits.device, "out")
        if idx is not None and (idx.dtype != torch.int32 or idx.numel() < n or not idx.is_contiguous()
                                or idx.device != hits.device):
            raise FiberError("compact_hits: idx must be a contiguous int32[>= n] on the hits' device")
        if count.dtype != torch.int32 or count.numel() < 1 or count.device != hits.device:
            raise FiberError("compact_hits: count must be int32[1] on the hits' device")
        _check(lib().fiber_compact_hits(hits.data_ptr(), n, out.data_ptr(),
                                        idx.data_ptr() if idx is not None else None,
                                        count.data_ptr(), _stream(stream)), "fiber_compact_hits")
    return out, idx, count


def nearest_init(nearest: torch.Tensor, stream=None) -> torch.Tensor:
    """fiber_nearest_init: every key to 'no hit' (all ones = -1 as int64)."""
    if not (isinstance(nearest, torch.Tensor) and nearest.is_cuda and nearest.dtype == torch.int64
            and nearest.is_contiguous()):
        raise FiberError("nearest must be a contiguous CUDA int64 tensor")
    _check(lib().fiber_nearest_init(nearest.data_ptr(), nearest.numel(), _stream(stream)),
           "fiber_nearest_init")
    return nearest


def nearest_records(nearest: torch.Tensor, hits: torch.Tensor, pairs: torch.Tensor,
                    ray_ids: torch.Tensor, out: torch.Tensor | None = None,
                    stream=None) -> torch.Tensor:
    """fiber_nearest_records: per-ray records (t, u, n_oct, segment; misses t = +inf, segment
    = -1) of the rays `ray_ids` from one nearest-hit launch's keys, records and pairs."""
    with _on(stream):
        pairs = _pairs(pairs)
        _hits(hits, pairs.shape[0], pairs.device)
        if not (nearest.is_cuda and nearest.dtype == torch.int64 and nearest.is_contiguous()):
            raise FiberError("nearest must be a contiguous CUDA int64 tensor")
        ray_ids = ray_ids.to(torch.int64).contiguous()
        if not ray_ids.is_cuda or ray_ids.device != pairs.device:
            raise FiberError("ray_ids must be a CUDA tensor on the pairs' device")
        n = ray_ids.numel()
        if out is None:
            out = torch.empty((n, 4), dtype=torch.float32, device=pairs.device)
        _hits(out, n, pairs.device, "out")
        _check(lib().fiber_nearest_records(nearest.data_ptr(), hits.data_ptr(), pairs.data_ptr(),
                                           ray_ids.data_ptr(), n, out.data_ptr(), _stream(stream)),
               "fiber_nearest_records")
    return out


# ------------------------------------------------------------------------- host helpers
def decode_normals(n_oct: np.ndarray) -> np.ndarray:
    """Vectorised octahedral snorm16x2 decode (same convention as fiber_decode_normal)."""
    n_oct = np.asarray(n_oct).view(np.uint32)
    x = (n_oct & 0xFFFF).astype(np.uint16).view(np.int16).astype(np.float64) / 32767.0
    y = (n_oct >> 16).astype(np.uint16).view(np.int16).astype(np.float64) / 32767.0
    z = 1.0 - np.abs(x) - np.abs(y)
    neg = z < 0
    ox = (1.0 - np.abs(y)) * np.where(x >= 0, 1.0, -1.0)
    oy = (1.0 - np.abs(x)) * np.where(y >= 0, 1.0, -1.0)
    x = np.where(neg, ox, x)
    y = np.where(neg, oy, y)
    v = np.stack([x, y, z], -1)
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def unpack(hits) -> dict:
    """hits f32[n,4] (torch or numpy) -> dict(t, u, n[n,3], flags, hit, kind, inside,
    bad_input, bad_segment, backtracks, tests) as numpy arrays."""
    h = hits.detach().cpu().numpy() if isinstance(hits, torch.Tensor) else np.asarray(hits)
    h = np.ascontiguousarray(h, dtype=np.float32)
    bits = h.view(np.uint32)
    flags = bits[:, 3]
    return {
        "t": h[:, 0].astype(np.float64), "u": h[:, 1].astype(np.float64),
        "n": decode_normals(bits[:, 2]), "flags": flags,
        "hit": (flags & HIT) != 0, "kind": ((flags >> KIND_SHIFT) & 3).astype(np.int32),
        "inside": (flags & INSIDE) != 0, "bad_input": (flags & BAD_INPUT) != 0,
        "bad_segment": (flags & BAD_SEGMENT) != 0,
        "backtracks": ((flags >> 8) & 0xFF).astype(np.int32),
        "tests": ((flags >> 16) & 0xFFFF).astype(np.int32),
    }


def pack_rays(rays_np: np.ndarray, device="cuda") -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(rays_np, dtype=np.float32)).to(device)


def to_device(workload, device="cuda"):
    """Move a workloads.gen.Workload to the GPU: (rays, Segments, pairs)."""
    rays = torch.from_numpy(np.ascontiguousarray(workload.rays)).to(device)
    ctrl = torch.from_numpy(np.ascontiguousarray(workload.ctrl)).to(device)
    radii = torch.from_numpy(np.ascontiguousarray(workload.radii)).to(device)
    pairs = torch.from_numpy(np.ascontiguousarray(workload.pairs).view(np.int32)).to(device)
    segs = (build_segments_quadratic if ctrl.shape[1] == 3 else build_segments)(ctrl, radii)
    return rays, segs, pairs

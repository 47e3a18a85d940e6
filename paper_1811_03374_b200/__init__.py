"""B200-native (sm_100a) ray/fiber intersection: Binder & Keller, arXiv 1811.03374.

The product path is libfiber.so (CUDA C ABI, include/fiber.h) behind the ctypes binding in
``fiber``; ``dist`` shards rays across GPUs.  There is no CPU fallback.
"""
from .fiber import (BAD_INPUT, BAD_SEGMENT, HIT, INSIDE, Grid, KIND_CAP0, KIND_CAP1, KIND_LATERAL,  # noqa: F401
                    KIND_WEDGE, MAX_DEPTH, FiberError, Segments, build_segments, build_segments_quadratic,
                    compact_hits, decode_normals,
                    intersect, intersect_closest, intersect_ex, intersect_nearest, lib, nearest_init,
                    nearest_records, presplit,
                    remap_u, to_device,
                    unpack)

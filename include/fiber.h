/*
 * fiber.h -- C ABI of the B200 (sm_100a) ray/fiber intersection library (libfiber.so).
 *
 * The operation is the one of Binder & Keller, "Fast, High Precision Ray/Fiber
 * Intersection using Tight, Disjoint Bounding Volumes" (arXiv 1811.03374): given a ray
 * (origin, direction, t_max) and a fiber -- a circular contour of cubic-Bezier radius swept
 * along a cubic Bezier curve -- return the nearest intersection (t, u, normal) or nothing
 * (lst:algorithm).  The method is the stackless
 * subdivision with disjoint bounding cylinders at a fixed depth D, with the
 * readings F1-F9 documented in DESIGN.md.
 *
 * Conventions for every call:
 *   - Pointers marked "device" are CUDA device pointers owned by the caller.  The library
 *     keeps, per device and per process, immutable launch constants and a private
 *     stream-ordered memory pool from which each fiber_intersect call takes its scratch
 *     (its own work counters, zeroed on its stream, and work lists: 256 B + 8 B per pair;
 *     16 B more per pair when no hits buffer is given) and returns it on the same stream.
 *     No state is shared between calls, so any number may be in flight on any streams.
 *     It is re-entrant and thread-safe.
 *   - Work is enqueued on `cuda_stream` (a cudaStream_t, NULL = legacy default stream) and
 *     the call returns immediately; outputs are valid after that stream synchronises, and
 *     inputs must not change before then.  Kernel faults surface at the next sync.
 *   - Return value: FIBER_OK, or a negative fiber_status.  Argument errors are detected
 *     before anything is enqueued.  Data errors (NaN, out-of-range indices, segments that
 *     violate the paper's constraints) never abort: they are reported per record in flags.
 */
#ifndef FIBER_H
#define FIBER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 23 mantissa bits hold the parametric interval (lst:calculate_interval P:1331-1345,
 * cur_size = 1 << 23 at P:1605): depth D in [0, 23], min_size = 2^(23 - D). */
#define FIBER_MAX_DEPTH 23

typedef enum {
  FIBER_OK = 0,
  FIBER_EINVAL = -1,  /* NULL pointer with n > 0, n < 0, n >= 2^32, depth not in [0, 23] */
  FIBER_ECUDA = -2,   /* a CUDA call or launch failed; see fiber_error_string()          */
  FIBER_EDEVICE = -3  /* the current device is not an sm_100 (B200) GPU                  */
} fiber_status;

/* A ray o + t d, t in [0, tmax) (unit ray of P:475-481; t_max of P:1610).
 * d need not be exactly unit: t is the parameter along d as given.  tmax may be +inf. */
typedef struct {
  float ox, oy, oz, tmax;
  float dx, dy, dz, pad;
} fiber_ray; /* 32 B */

/* One ray-segment candidate (the unit of work; produced by a top-level hierarchy). */
typedef struct {
  uint32_t ray, seg;
} fiber_pair; /* 8 B */

/* Per-pair result (lst:calc_intersection P:1546-1587).
 *   t      ray parameter of the hit (+inf on a miss)
 *   u      curve parameter in [0, 1] (0 on a miss)
 *   n_oct  unit surface normal, octahedral encoding, 2 x snorm16 (x in bits 0-15,
 *          y in bits 16-31); see fiber_decode_normal().  0 on a miss.
 *   flags  FIBER_HIT, kind (bits 1-2), FIBER_INSIDE, FIBER_BAD_INPUT, FIBER_BAD_SEGMENT,
 *          backtracks (bits 8-15, saturating), node tests (bits 16-31, saturating). */
typedef struct {
  float t, u;
  uint32_t n_oct, flags;
} fiber_hit; /* 16 B */

#define FIBER_HIT (1u << 0)
#define FIBER_KIND_SHIFT 1
#define FIBER_KIND_MASK (3u << 1)
#define FIBER_KIND_LATERAL 0u /* entry through the lateral surface                       */
#define FIBER_KIND_CAP0 1u    /* entry through the start cap, u = 0 (F6)     */
#define FIBER_KIND_CAP1 2u    /* entry through the end cap,   u = 1                       */
#define FIBER_KIND_WEDGE 3u   /* entry through an internal partition plane (low D, F2)   */
#define FIBER_INSIDE (1u << 3)      /* ray origin inside the fiber: t = 0                   */
#define FIBER_BAD_INPUT (1u << 4)   /* non-finite ray, zero direction, tmax <= 0, or an index
                                       out of range: the record is a miss                   */
#define FIBER_BAD_SEGMENT (1u << 5) /* the segment failed fiber_build_segments' checks; the
                                       pair is still computed but the result is unspecified
                                                                                 */
#define FIBER_BACKTRACKS(f) (((f) >> 8) & 0xffu)
#define FIBER_NODE_TESTS(f) (((f) >> 16) & 0xffffu)

/* Segment flags written by fiber_build_segments (0 = valid). */
#define FIBER_SEG_CONSTRAINT(k) (1u << (k)) /* k = 0..4: the k-th cubic inequality of
                                               P:614-621 fails (App. B eqs)    */
#define FIBER_SEG_DEGENERATE (1u << 5)      /* zero chord or an end tangent shorter than
                                               1e-6 of the chord (plane normal undefined)   */
#define FIBER_SEG_NONFINITE (1u << 6)       /* a NaN/Inf coordinate or radius             */
#define FIBER_SEG_NEG_RADIUS (1u << 7)      /* a negative radius                           */
#define FIBER_SEG_QUADRATIC (1u << 8)       /* not an error: a quadratic segment (written by
                                               fiber_build_segments_quadratic); its planes hold
                                               p0 = q0, p1 = p2 = q1, p3 = q2 and the kernels
                                               degree-elevate it exactly (App. B.1)     */
#define FIBER_SEG_QUAD_CONSTRAINT (1u << 9) /* the quadratic constraint
                                               <q1 - q0, q1 - q2> <= 0 (App. B.1 eq. P:889) fails */
#define FIBER_SEG_THICK (1u << 10)          /* advisory: with the largest radius control point
                                               r_bar the surface would cross an end plane
                                               (the conservative test of P:686, "or just")    */
#define FIBER_SEG_THICK_PARAM (1u << 11)    /* the surface with the cubic radius r(u) crosses
                                               an end plane: a valid part of
                                               the fiber would be cropped (thick fiber / cusp) */
/* Bits that make a segment invalid (FIBER_BAD_SEGMENT on its pairs). */
#define FIBER_SEG_INVALID_MASK (~(FIBER_SEG_QUADRATIC | FIBER_SEG_THICK))

/* Device-resident segment set, structure of arrays: p[i][s] = (x, y, z, r) of control
 * point i of segment s, one float4 plane per control point (16-B aligned, coalesced
 * float4 loads).  A host-side descriptor of caller-owned device storage. */
typedef struct {
  void *p0, *p1, *p2, *p3; /* device float4[n]            */
  uint32_t *flags;         /* device uint32[n], 0 = valid */
  int64_t n;
} fiber_segments;

/* Bytes of device storage needed for n segments (4 float4 planes + flags, 256-B aligned). */
size_t fiber_segments_bytes(int64_t n);

/* Host-only: carve `storage` (device, >= fiber_segments_bytes(n) bytes, 256-B aligned)
 * into the SoA planes of `out`.  No device work. */
int fiber_segments_view(void *storage, int64_t n, fiber_segments *out);

/* Segment preprocessing: pack control points and radii into the SoA
 * planes of `segs` and validate each segment (the five cubic constraints of P:614-621,
 * degenerate tangents, non-finite values, negative radii) into segs->flags.
 *   ctrl_pts  device float[n][4][3]  control point positions (the 4-D control points of
 *                                    P:485-486 without the radius)
 *   radii     device float[n][4]     radius at each control point (cubic radius)
 *   segs      in: a view of n segments (fiber_segments_view); out: filled on device
 * Errors: FIBER_EINVAL (NULL with n > 0, n < 0, n >= 2^32, segs->n != n),
 *         FIBER_EDEVICE, FIBER_ECUDA. */
int fiber_build_segments(const float *ctrl_pts, const float *radii, int64_t n,
                         fiber_segments *segs, void *cuda_stream);

/* Quadratic fibers (the paper evaluates quadratic and cubic fibers,
 * P:707): like fiber_build_segments for quadratic Bezier segments.  The segment is stored
 * unrounded (p0 = q0, p1 = p2 = q1, p3 = q2, flag FIBER_SEG_QUADRATIC) and every kernel uses
 * its exact degree elevation (q0, (q0 + 2 q1)/3, (2 q1 + q2)/3, q2) -- the same curve and
 * radius function -- so the cubic method applies unchanged (de Casteljau halving commutes
 * with elevation).  The App. B.1 constraint (eq. P:889) implies the five cubic ones for the
 * elevated curve; it is checked into FIBER_SEG_QUAD_CONSTRAINT.
 *   ctrl_pts  device float[n][3][3]  control point positions q0, q1, q2
 *   radii     device float[n][3]     radius at each control point (quadratic radius)
 * A segment set is either all cubic or all quadratic.  Errors as fiber_build_segments. */
int fiber_build_segments_quadratic(const float *ctrl_pts, const float *radii, int64_t n,
                                   fiber_segments *segs, void *cuda_stream);

/* Input gatekeeper, pre-splitting (3.4 P:609-703: curves that violate the
 * constraints, and thick or cusp-like regions, "must be subdivided beforehand").  Every
 * cubic segment is bisected at the parameter midpoint (de Casteljau, FP64) until each piece
 * satisfies the five constraints and neither of its end planes is crossed by
 * its surface (the thick-fiber test: r = r(u) if parametric, else the largest radius
 * control point), or max_level halvings are reached.  Pieces tile [0, 1] in curve order.
 * Two calls: _count writes offsets (device uint32[n + 1]; offsets[s] = first piece of
 * segment s, offsets[n] = total, valid after the stream syncs); _write then fills
 *   out_ctrl  device float[total][4][3], out_radii device float[total][4] (FP32-rounded
 *             FP64 sub-curves; feed to fiber_build_segments),
 *   out_src   device uint32[total]  source segment,
 *   out_u     device float[total][2] (u0, u1) of the piece on its source (dyadic, exact),
 *   out_valid device uint32[total]  1 if the piece passes, 0 if max_level was reached.
 * max_level in [0, 16].  Errors: FIBER_EINVAL, FIBER_EDEVICE, FIBER_ECUDA. */
int fiber_presplit_count(const float *ctrl_pts, const float *radii, int64_t n, int max_level,
                         int parametric, uint32_t *offsets, void *cuda_stream);
int fiber_presplit_write(const float *ctrl_pts, const float *radii, int64_t n, int max_level,
                         int parametric, const uint32_t *offsets, float *out_ctrl,
                         float *out_radii, uint32_t *out_src, float *out_u, uint32_t *out_valid,
                         void *cuda_stream);

/* u remapping after intersecting pre-split pieces: for every hit record whose pair names
 * piece k, u <- u0[k] + u (u1[k] - u0[k]) (out_u of fiber_presplit_write); a cap kind at an
 * inner piece boundary (u0 > 0 for CAP0, u1 < 1 for CAP1) becomes WEDGE (an internal plane).
 *   hits device fiber_hit[n_pairs] (in/out), pairs device fiber_pair[n_pairs],
 *   piece_u device float[n_pieces][2].  Errors: FIBER_EINVAL, FIBER_EDEVICE, FIBER_ECUDA. */
int fiber_remap_u(fiber_hit *hits, const fiber_pair *pairs, int64_t n_pairs, const float *piece_u,
                  int64_t n_pieces, void *cuda_stream);

/* Candidate-pair generation (the top-level hierarchy of P:753-759): a
 * uniform grid over the segments' bounding boxes (control points dilated by the largest
 * radius control point) and a 3-D DDA per ray that emits every segment whose box
 * the ray overlaps on [0, tmax), front to back by cell (ascending segment id within a cell).
 * Conservative: a segment the ray hits is always a candidate (boxes are dilated by 1e-3 of a
 * cell against FP32 rounding; a segment may appear twice, which does not change a nearest
 * hit).  The grid is an opaque handle that owns its device memory. */
typedef struct fiber_grid_s fiber_grid;

/* Build the grid over `segs` (about cells_per_segment x n cells, each axis <= 1024) on the
 * current device.  Synchronises the stream (the sizes are data-dependent).
 * Errors: FIBER_EINVAL (n == 0, NULL, cells_per_segment <= 0), FIBER_EDEVICE, FIBER_ECUDA. */
int fiber_grid_create(const fiber_segments *segs, float cells_per_segment, fiber_grid **grid,
                      void *cuda_stream);
int fiber_grid_destroy(fiber_grid *grid);
/* Host-only: cells per axis and the number of (cell, segment) entries. */
int fiber_grid_info(const fiber_grid *grid, int32_t dims[3], int64_t *n_entries);

/* Pass 1: offsets (device uint32[n_rays + 1]) = exclusive scan of the candidate counts per
 * ray; *max_count and *total (host) are the largest count and offsets[n_rays].  Synchronises
 * the stream. */
int fiber_grid_count(const fiber_grid *grid, const fiber_ray *rays, int64_t n_rays,
                     uint32_t *offsets, uint32_t *max_count, uint64_t *total, void *cuda_stream);

/* Pass 2: write the total candidate pairs into pairs (device fiber_pair[total]).
 *   order 0: ray-major (ray r's candidates at offsets[r] .. offsets[r+1], front to back);
 *   order 1: rounds (every ray's first candidate in ray order, then every second one, ...),
 *            the order fiber_intersect_closest prunes best with (deterministic).
 * Errors: FIBER_EINVAL, FIBER_EDEVICE, FIBER_ECUDA. */
int fiber_grid_candidates(const fiber_grid *grid, const fiber_ray *rays, int64_t n_rays,
                          const uint32_t *offsets, uint32_t max_count, int order,
                          fiber_pair *pairs, void *cuda_stream);

/* Closest hit over the grid's candidates with early termination (SURVEY 8(f) rows 2 + 3):
 * rounds of (walk: each active ray's DDA emits its next k candidates, k = 8, 16, ... 256;
 * fiber_intersect_closest on them) until every ray's walk is over or its best hit lies
 * strictly before the walk's position -- exact, since a later candidate enters its box at or
 * after that position and its hits lie in the box.
 *   nearest  device uint64[n_rays], initialised by the caller (fiber_nearest_init); on return
 *            nearest[r] = min over r's candidates of (bits(t) << 32) | segment index -- keys
 *            carry the SEGMENT (not a pair index), so the result does not depend on the order
 *            of the rounds.
 *   rounds   (host, may be NULL) the number of rounds run.
 * Synchronises the stream once per round.  Errors: FIBER_EINVAL, FIBER_EDEVICE, FIBER_ECUDA. */
int fiber_grid_closest(const fiber_grid *grid, const fiber_ray *rays, int64_t n_rays,
                       const fiber_segments *segs, int max_depth, uint64_t *nearest,
                       int *rounds, void *cuda_stream);

/* The hot path (lst:algorithm): for every pair, intersect rays[pair.ray] with
 * segment pair.seg at subdivision depth max_depth and write hits[i].
 *   rays      device fiber_ray[n_rays]
 *   segs      built by fiber_build_segments (host descriptor, device planes)
 *   pairs     device fiber_pair[n_pairs], 0 <= n_pairs < 2^31 (a larger set takes several
 *             calls); indices out of range give FIBER_BAD_INPUT
 *   max_depth D in [0, 23]: the number of halvings of [0, 1]; min_size = 2^(23 - D)
 *   hits      device fiber_hit[n_pairs]
 * Results are bit-identical for the same inputs regardless of launch shape or order.
 * Errors: FIBER_EINVAL (also n_pairs >= 2^31, n_rays >= 2^32), FIBER_EDEVICE, FIBER_ECUDA. */
int fiber_intersect(const fiber_ray *rays, int64_t n_rays, const fiber_segments *segs,
                    const fiber_pair *pairs, int64_t n_pairs, int max_depth, fiber_hit *hits,
                    void *cuda_stream);

/* fiber_intersect with the per-ray nearest-hit epilogue: in addition
 * (hits may be NULL), for every hit pair atomically
 *   nearest[pair.ray] = min(nearest[pair.ray], (bits(t) << 32) | i)
 * where i is the pair index in this call.  `nearest` (device uint64[n_rays]) must be
 * initialised by the caller (fiber_nearest_init) before the first call of a batch.  The keys
 * are formed by a pass over the finished records queued after the traversal on the same
 * stream (the result is the same min as forming them at each hit). */
int fiber_intersect_nearest(const fiber_ray *rays, int64_t n_rays, const fiber_segments *segs,
                            const fiber_pair *pairs, int64_t n_pairs, int max_depth,
                            fiber_hit *hits, uint64_t *nearest, void *cuda_stream);

/* Closest hit over candidate lists: fiber_intersect_nearest where each
 * pair's traversal is bounded by the best hit its ray has so far -- the ray's t_max used as a
 * running bound: when a pair starts, t_max' = min(ray.tmax, t_best (1 + 2^-19)),
 * t_best read from nearest[pair.ray].  A bounded traversal returns the unbounded first hit
 * whenever that lies before the bound, and a miss otherwise, so `nearest` ends bit-identical
 * to fiber_intersect_nearest's; pairs are only pruned sooner.  The pruning depends on the
 * order: give each ray's candidates in rounds, nearest candidates first (all rays' first
 * candidate, then all second candidates, ...).  hits (may be NULL) holds every pair's record,
 * but only the winning pair's record of each ray is defined (a pair behind the running bound
 * reads as a miss).  Errors as fiber_intersect_nearest. */
int fiber_intersect_closest(const fiber_ray *rays, int64_t n_rays, const fiber_segments *segs,
                            const fiber_pair *pairs, int64_t n_pairs, int max_depth,
                            fiber_hit *hits, uint64_t *nearest, void *cuda_stream);

/* fiber_intersect / fiber_intersect_nearest in one call (hits or nearest may be NULL, not
 * both), for callers that time the stages: when event_after_traverse (a cudaEvent_t) is
 * not NULL it is recorded on the stream between the traversal kernel (K2, SURVEY 8(a)
 * a2-a6) and the finalisation kernel (K3, a7: FP64 re-runs of near-tie pairs and FP64
 * re-solves of hits that need them).  Errors as fiber_intersect. */
int fiber_intersect_ex(const fiber_ray *rays, int64_t n_rays, const fiber_segments *segs,
                       const fiber_pair *pairs, int64_t n_pairs, int max_depth, fiber_hit *hits,
                       uint64_t *nearest, void *event_after_traverse, void *cuda_stream);

/* Order-preserving stream compaction of hit records, for callers that move only the hits
 * off the device (the problem statement returns "the nearest intersection or nothing",
 * P:251-257, so a pair without FIBER_HIT carries no result).
 *   hits   device fiber_hit[n], as written by fiber_intersect / _ex (complete: call after them
 *          on the same stream)
 *   n      number of records, 0 <= n < 2^32
 *   out    device fiber_hit[n] (worst case): out[k] = hits[idx[k]], k < *count
 *   idx    device uint32[n] or NULL: idx[k] = the pair index of the k-th hit, increasing
 *   count  device uint32[1]: the number of records with FIBER_HIT
 * Deterministic (the k-th hit in pair order goes to slot k).  Scratch comes from the
 * library's stream-ordered pool.  Asynchronous like fiber_intersect.
 * Errors: FIBER_EINVAL (n out of range, count NULL, hits/out NULL with n > 0),
 * FIBER_EDEVICE, FIBER_ECUDA. */
int fiber_compact_hits(const fiber_hit *hits, int64_t n, fiber_hit *out, uint32_t *idx,
                       uint32_t *count, void *cuda_stream);

/* Fill nearest[0..n_rays) with the "no hit" key (all ones). */
int fiber_nearest_init(uint64_t *nearest, int64_t n_rays, void *cuda_stream);

/* Per-ray records of the nearest-hit epilogue (the records a multi-GPU
 * run gathers, 16 B per ray).  For j in [0, n): r = ray_ids[j], key = nearest[r] (as written by
 * fiber_intersect_nearest over `pairs` / `hits` of ONE launch, the key's low word is the pair
 * index in it):
 *   key == all ones (no hit): out[j] = {t = +inf, u = 0, n_oct = 0, flags = 0xffffffff}
 *   else i = key & 0xffffffff: out[j] = {hits[i].t, hits[i].u, hits[i].n_oct, pairs[i].seg}
 * i.e. the record of the ray's first hit with the hit segment's index in place of the flags.
 *   nearest  device uint64[>= max ray id + 1];  hits, pairs  device, of the launch
 *   ray_ids  device int64[n];  out  device fiber_hit[n] (may not alias the inputs)
 * Errors: FIBER_EINVAL (n < 0, NULL with n > 0), FIBER_EDEVICE, FIBER_ECUDA. */
int fiber_nearest_records(const uint64_t *nearest, const fiber_hit *hits, const fiber_pair *pairs,
                          const int64_t *ray_ids, int64_t n, fiber_hit *out, void *cuda_stream);

/* Static description of the last failure on this thread (or of `code`). */
const char *fiber_error_string(int code);

/* Host helper: decode an octahedral snorm16x2 normal into out[3] (unit length). */
void fiber_decode_normal(uint32_t n_oct, float out[3]);

/* ABI version (major * 100 + minor). */
int fiber_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FIBER_H */

// intersect.cu -- K2: the ray/fiber pair intersector for sm_100a, plus its C ABI.
//
// One thread per ray-segment pair, the stackless traversal of
// lst:algorithm with the readings F1-F9 of DESIGN.md.
// DESIGN.md "Kernel" describes the launch shape and precision split.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <atomic>
#include <chrono>
#include <unistd.h>
#include <mutex>

#include "fiber.h"
#include "exact.cuh"
#include "fiber_device.cuh"
#include "fiber_internal.h"

namespace fiberx {

#ifndef FIBER_K2_THREADS
#define FIBER_K2_THREADS 256
#endif
#ifndef FIBER_FAR_CACHE
#define FIBER_FAR_CACHE 2
#endif
constexpr int kThreads = FIBER_K2_THREADS;
constexpr int kWarps = kThreads / 32;
constexpr int kFarCache = FIBER_FAR_CACHE;  // per-lane cache of pending far children
constexpr int kRingF4 = 5;  // a ring entry: the parent's Delta (4 float4) + its interval
constexpr int kRayStash = 1;  // per-lane copy of the ray direction + ray index (end_pair)
constexpr size_t kSmemBytes = (size_t)(4 + kRingF4 * kFarCache + kRayStash) * kThreads * sizeof(float4) +
                               kThreads * sizeof(uint32_t);  // + the lanes' FP64 resume points

// ------------------------------------------------------------------------------------
// a7: FP64 finalisation (lst:calc_intersection P:1546-1587 with F2, F6, F8)
// ------------------------------------------------------------------------------------
// World coordinates relative to the segment anchor c = fl((P0 + P3)/2): every input is an
// FP32 number, so differences are exact or nearly so in FP64 and no frame is needed.
struct D4 {
  double x, y, z, w;
};
__device__ __forceinline__ D4 d4of(float4 a) { return D4{a.x, a.y, a.z, a.w}; }
__device__ __forceinline__ D4 dsub(D4 a, D4 b) { return D4{a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w}; }
__device__ __forceinline__ D4 dadd(D4 a, D4 b) { return D4{a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w}; }
__device__ __forceinline__ D4 dscale(double s, D4 a) { return D4{s * a.x, s * a.y, s * a.z, s * a.w}; }
__device__ __forceinline__ double ddot3(D4 a, D4 b) { return fma(a.x, b.x, fma(a.y, b.y, a.z * b.z)); }
__device__ __forceinline__ D4 dcross(D4 a, D4 b) {
  return D4{fma(a.y, b.z, -a.z * b.y), fma(a.z, b.x, -a.x * b.z), fma(a.x, b.y, -a.y * b.x), 0.0};
}

struct LeafD {
  D4 p, d, t0, t1;  // (p, d, t0, t1) form of 3.1, relative to the anchor
};

// Sub-curve on [u0, u1] from the hodograph blossoms (as recompute(), in FP64).
__device__ __forceinline__ LeafD leaf_d(D4 q0, D4 D0, D4 D1, D4 D2, double u0, double u1) {
  auto H = [&](double a, double b) {
    double wa = (1.0 - a) * (1.0 - b), wb = a * (1.0 - b) + (1.0 - a) * b, wc = a * b;
    return D4{fma(wa, D0.x, fma(wb, D1.x, wc * D2.x)), fma(wa, D0.y, fma(wb, D1.y, wc * D2.y)),
              fma(wa, D0.z, fma(wb, D1.z, wc * D2.z)), fma(wa, D0.w, fma(wb, D1.w, wc * D2.w))};
  };
  double h = u1 - u0;
  D4 H00 = H(u0, u0), H01 = H(u0, u1), H11 = H(u1, u1), H0u = H(0.0, u0);
  D4 s = dadd(dadd(D0, H0u), H00);
  LeafD q;
  q.p = D4{fma(u0, s.x, q0.x), fma(u0, s.y, q0.y), fma(u0, s.z, q0.z), fma(u0, s.w, q0.w)};
  q.t0 = dscale(h, H00);
  q.t1 = dscale(h, H11);
  q.d = dscale(h, dadd(dadd(H00, H01), H11));
  return q;
}

// Entry parameter t of the ray m + t w (m relative to the anchor) into the infinite
// conservative cylinder of leaf q, FP64, in App. A's closest-approach form
// (d^2 of eq. P:814, t_cpa P:825-833, s P:862-866) with n = w x d, which keeps full
// precision near tangency (the expanded quadratic would cancel).
__device__ __forceinline__ bool leaf_entry(const LeafD& q, D4 m, D4 w, double& t,
                                           double* t_exit = nullptr) {
  double dd = ddot3(q.d, q.d);
  D4 x0 = dcross(q.t0, q.d), x1 = dcross(q.t1, q.d);
  double m2 = fmax(ddot3(x0, x0), ddot3(x1, x1));
  double maxr = q.p.w + fmax(fmax(0.0, q.t0.w), fmax(q.d.w, q.d.w - q.t1.w));
  double R = exact::sqrt64(m2 * exact::rcp64(dd)) + maxr;
  D4 mm = dsub(m, q.p);
  D4 n = dcross(w, q.d);            // |n|^2 = |w x d|^2
  double A = ddot3(n, n);
  if (!(A > 0.0)) return false;
  double mn = ddot3(mm, n);
  const double iA = exact::rcp64(A);
  double d2 = mn * mn * iA;         // squared line-line distance (eq. P:814)
  if (!(d2 <= R * R)) return false;
  D4 md = dcross(mm, q.d);
  double tcpa = -ddot3(md, n) * iA;
  const double hs = exact::sqrt64((R * R - d2) * dd * iA);
  t = tcpa - hs;
  if (t_exit) *t_exit = tcpa + hs;
  return isfinite(t);
}

// Octahedral snorm16x2 encoding of a (not necessarily unit) FP32 direction.
__device__ __forceinline__ uint32_t encode_oct_f(float x, float y, float z) {
  const float l1 = fabsf(x) + fabsf(y) + fabsf(z);
  if (!(l1 > 0.0f)) return 0u;
  const float il = frcp(l1);
  x *= il;
  y *= il;
  if (z < 0.0f) {
    const float ox = (1.0f - fabsf(y)) * copysignf(1.0f, x);
    const float oy = (1.0f - fabsf(x)) * copysignf(1.0f, y);
    x = ox;
    y = oy;
  }
  const int ix = __float2int_rn(fminf(1.0f, fmaxf(-1.0f, x)) * 32767.0f);
  const int iy = __float2int_rn(fminf(1.0f, fmaxf(-1.0f, y)) * 32767.0f);
  return ((uint32_t)ix & 0xffffu) | (((uint32_t)iy & 0xffffu) << 16);
}

__device__ __forceinline__ uint32_t encode_oct32(double nx, double ny, double nz) {
  double mx = fmax(fabs(nx), fmax(fabs(ny), fabs(nz)));
  if (!(mx > 0.0)) return 0u;
  float x = (float)(nx / mx), y = (float)(ny / mx), z = (float)(nz / mx);
  float l1 = fabsf(x) + fabsf(y) + fabsf(z);
  x /= l1;
  y /= l1;
  if (z < 0.0f) {
    float ox = (1.0f - fabsf(y)) * copysignf(1.0f, x);
    float oy = (1.0f - fabsf(x)) * copysignf(1.0f, y);
    x = ox;
    y = oy;
  }
  int ix = __float2int_rn(fminf(1.0f, fmaxf(-1.0f, x)) * 32767.0f);
  int iy = __float2int_rn(fminf(1.0f, fmaxf(-1.0f, y)) * 32767.0f);
  return ((uint32_t)ix & 0xffffu) | (((uint32_t)iy & 0xffffu) << 16);
}

// Re-solves the accepted leaf in FP64.  Lateral entries walk to the neighbouring leaf whose
// own slab holds the entry point (the FP32 leaf can be a few leaves off at D >= 16, where
// leaves are narrower than FP32 resolution); cap and crop-plane (WEDGE) entries re-solve
// the plane that bounds t_min; inside entries keep t = 0.
__device__ __forceinline__ void finalize(const float4 ray0, const float4 ray1, const float4 P0,
                                         const float4 P1, const float4 P2, const float4 P3,
                                         bool quad, uint32_t start, int depth, uint32_t kind,
                                         uint32_t lo_tag, float t32, int walk, float& t_out,
                                         float& u_out, uint32_t& n_out, bool& hit,
                                         uint32_t& kind_out) {
  kind_out = kind;
  const D4 c = D4{0.5 * ((double)P0.x + (double)P3.x), 0.5 * ((double)P0.y + (double)P3.y),
                  0.5 * ((double)P0.z + (double)P3.z), 0.0};
  const D4 q0 = dsub(d4of(P0), c);
  D4 D0 = dsub(d4of(P1), d4of(P0)), D1 = dsub(d4of(P2), d4of(P1)), D2 = dsub(d4of(P3), d4of(P2));
  if (quad) {  // exact degree elevation of (q0, q1, q2) = (P0, P1, P3), in FP64
    const D4 a = D0, b = dsub(d4of(P3), d4of(P1));
    D0 = dscale(2.0 / 3.0, a);
    D1 = dscale(1.0 / 3.0, dadd(a, b));
    D2 = dscale(2.0 / 3.0, b);
  }
  const D4 m = D4{(double)ray0.x - c.x, (double)ray0.y - c.y, (double)ray0.z - c.z, 0.0};
  const D4 w = D4{ray1.x, ray1.y, ray1.z, 0.0};
  const int64_t nleaf = (int64_t)1 << depth;
  const double inv = ldexp(1.0, -depth);
  int64_t k = (int64_t)(start >> (FIBER_MAX_DEPTH - depth));
  FIBER_CHECK(depth >= 0 && depth <= FIBER_MAX_DEPTH && k >= 0 && k < nleaf);
  double t = (double)t32, u = 0.0;
  D4 n;
  if (kind == FIBER_KIND_CAP0 || kind == FIBER_KIND_CAP1) {
    // the global cap plane of lst:calc_t_interval at u = 0 / u = 1, cap normal P:1567-1573
    bool c0k = kind == FIBER_KIND_CAP0;
    D4 qp = c0k ? q0 : dsub(d4of(P3), c);
    D4 nn = c0k ? D0 : D2;
    double wn = ddot3(w, nn);
    if (wn != 0.0) t = exact::div64(ddot3(dsub(qp, m), nn), wn);
    u = c0k ? 0.0 : 1.0;
    n = c0k ? dscale(-1.0, D0) : D2;
  } else {
    LeafD q = leaf_d(q0, D0, D1, D2, k * inv, (k + 1) * inv);
    if (kind == FIBER_KIND_WEDGE && lo_tag != TAG_ORIGIN) {
      // entry through the crop plane that bounds t_min: the normal plane at u = lo_tag
      // (through C(u), normal C'(u)/3 = H(u, u)), solved in FP64
      double ul = (double)lo_tag * (1.0 / (double)(1u << FIBER_MAX_DEPTH));
      LeafD pl = leaf_d(q0, D0, D1, D2, ul, ul + inv);  // p = C(ul), t0 = h H(ul, ul)
      double wn = ddot3(w, pl.t0);
      if (wn != 0.0) t = exact::div64(ddot3(dsub(pl.p, m), pl.t0), wn);
    }
    if (kind == FIBER_KIND_LATERAL) {
      // The leaf test of the oracle in FP64 (P:1618 with F1, F2): the infinite cylinder
      // interval of leaf kk against its own slab and [0, t_max); t* = max(c0, lo).
      const uint32_t sh = FIBER_MAX_DEPTH - depth;
      auto test = [&](int64_t kk, LeafD& qq, double& ts, uint32_t& lu, bool& lateral) {
        qq = leaf_d(q0, D0, D1, D2, kk * inv, (kk + 1) * inv);
        double c0, c1;
        if (!leaf_entry(qq, m, w, c0, &c1)) return false;
        double lo = 0.0, hi = (double)ray0.w;
        lu = TAG_ORIGIN;
        auto clip = [&](double alpha, double beta, uint32_t uu) {  // alpha + beta t >= 0
          if (beta > 0.0) {
            double x = exact::div64(-alpha, beta);
            if (x > lo) lo = x, lu = uu;
          } else if (beta < 0.0) {
            hi = fmin(hi, exact::div64(-alpha, beta));
          } else if (alpha < 0.0) {
            lo = INFINITY;
          }
        };
        const D4 mp = dsub(m, qq.p);
        clip(ddot3(mp, qq.t0), ddot3(w, qq.t0), (uint32_t)kk << sh);
        clip(-ddot3(dsub(mp, qq.d), qq.t1), -ddot3(w, qq.t1), (uint32_t)(kk + 1) << sh);
        lateral = c0 >= lo;
        ts = fmax(c0, lo);
        return (c1 >= lo) && (c0 <= hi) && (lo <= hi) && (ts < (double)ray0.w);
      };
      double ts;
      uint32_t lu;
      bool lat;
      bool ok = test(k, q, ts, lu, lat);
      int dir = 0;
      for (int it = 0; it < walk; ++it) {
        LeafD qn;
        double tn;
        uint32_t ln;
        bool latn;
        if (ok) {
          if (lat || lu == TAG_ORIGIN) break;  // a lateral entry inside the own slab: first
          // entered through a crop plane: the leaf across that plane may be entered earlier
          const int step = (lu == ((uint32_t)k << sh)) ? -1 : +1;
          if (k + step < 0 || k + step >= nleaf) break;
          if (!test(k + step, qn, tn, ln, latn) || !(tn < ts)) break;
          k += step;
          FIBER_CHECK(k >= 0 && k < nleaf);
        } else {
          // the FP32 leaf is off (below the crop level): walk towards the cylinder entry
          double c0;
          if (!leaf_entry(q, m, w, c0)) break;
          D4 X = dsub(D4{fma(c0, w.x, m.x), fma(c0, w.y, m.y), fma(c0, w.z, m.z), 0.0}, q.p);
          int step = 0;
          if (ddot3(X, q.t0) < 0.0 && k > 0 && dir <= 0) step = -1;
          else if (ddot3(dsub(X, q.d), q.t1) > 0.0 && k < nleaf - 1 && dir >= 0) step = +1;
          if (step == 0) break;
          dir = step;
          k += step;
          FIBER_CHECK(k >= 0 && k < nleaf);
          ok = test(k, qn, tn, ln, latn);
          if (!ok) {  // keep walking from the new leaf's geometry
            q = qn;
            continue;
          }
        }
        q = qn;
        ts = tn;
        lu = ln;
        lat = latn;
        ok = true;
      }
      if (!ok) {
        if (walk == 0) {  // an exact leaf that fails only by rounding: keep the FP32 entry
          double c0;
          if (leaf_entry(q, m, w, c0)) ts = c0, lat = true, ok = true;
        }
        if (!ok) {  // no leaf holds an entry: not a hit of the fiber
          hit = false;
          t_out = INFINITY;
          u_out = 0.0f;
          n_out = 0u;
          return;
        }
      }
      t = ts;
      if (!lat) {  // entry through a crop plane (WEDGE; the caps at u = 0 and u = 1)
        if (lu == TAG_ORIGIN) kind = FIBER_KIND_WEDGE;
        else if (lu == 0u) kind = FIBER_KIND_CAP0;
        else if (lu == (1u << FIBER_MAX_DEPTH)) kind = FIBER_KIND_CAP1;
        else kind = FIBER_KIND_WEDGE;
        kind_out = kind;
        if (kind == FIBER_KIND_CAP0 || kind == FIBER_KIND_CAP1) {  // cap normal
          const bool c0k = kind == FIBER_KIND_CAP0;
          n = c0k ? dscale(-1.0, D0) : D2;
          u = c0k ? 0.0 : 1.0;
          hit = t < (double)ray0.w;
          t_out = hit ? (float)t : INFINITY;
          u_out = hit ? (float)u : 0.0f;
          n_out = hit ? encode_oct32(n.x, n.y, n.z) : 0u;
          return;
        }
      }
    }
    // u by projection onto the leaf chord, normal from the axis point (F8)
    D4 X = dsub(D4{fma(t, w.x, m.x), fma(t, w.y, m.y), fma(t, w.z, m.z), 0.0}, q.p);
    double ul = exact::div64(ddot3(X, q.d), ddot3(q.d, q.d));
    ul = fmin(1.0, fmax(0.0, ul));
    u = ((double)k + ul) * inv;
    n = D4{fma(-ul, q.d.x, X.x), fma(-ul, q.d.y, X.y), fma(-ul, q.d.z, X.z), 0.0};
  }
  hit = t < (double)ray0.w;
  t_out = hit ? (float)t : INFINITY;
  u_out = hit ? (float)u : 0.0f;
  n_out = hit ? encode_oct32(n.x, n.y, n.z) : 0u;
}

// ------------------------------------------------------------------------------------
// a2 setup: FP32 frame with an FP64-exact origin shift
// ------------------------------------------------------------------------------------
// The frame origin o' = o + ts d is placed on the ray next to the segment anchor
// c = fl((P0 + P3) / 2) (ts: the ray parameter along d as given).  With w^ = d / |d| (FP32,
// ~1 ulp) and (b1, b2) the FP32 Duff/Frisvad basis of w^, local coordinates of
// a point X are (<X-o', b1>, <X-o', b2>, <X-o', w^>).  They are split as <X - c, b> (small,
// FP32) + rho, rho = <c - o - ts d, b>: rho carries the cancellation of |c - o| ~ |ray
// length| and is formed in FP64 from the exact FP32 inputs, so every local coordinate is
// accurate to FP32 rounding of the SEGMENT's size.  The ray is then the unit ray
// (0,0,0) + z (0,0,1) of P:475-481 with z = (t - ts) |d|; t = (z - lo0) / |d|, lo0 = -ts |d|.
struct Setup32 {
  float4 b1, b2, wh;  // xyz used
  float ts, iw, lw;   // ts; 1 / |d|; |d|
};

// the ONB (b1, b2) of a unit direction (Duff et al.)
__device__ __forceinline__ void onb(const float4 wh, float4& b1, float4& b2) {
  const float sign = copysignf(1.0f, wh.z);
  const float a = -frcp(sign + wh.z);  // (1 ulp; the basis only needs orthonormality to ~1e-7)
  const float b = wh.x * wh.y * a;
  b1 = make_float4(fmaf(sign * wh.x * wh.x, a, 1.0f), sign * b, -sign * wh.x, 0.0f);
  b2 = make_float4(b, fmaf(wh.y * wh.y, a, sign), -wh.y, 0.0f);
}

// |d|^2 within 2^-22 of 1: unit to FP32 rounding (the SPEC contract S:34; every normalised
// FP32 vector).  K2 traverses only such rays, in the frame of w^ = d as is;
// any other d is traversed by K3 in FP64 (exact.cuh normalises it), t along d as given.
__device__ __forceinline__ bool unit_dir(float ww) {
  return fabsf(ww - 1.0f) <= 2.384185791015625e-07f;
}

// kUnit: the caller has checked unit_dir (K2); otherwise d is normalised (K3's finalisation)
template <bool kUnit>
__device__ __forceinline__ bool frame32(const float4 ray0, const float4 ray1, const float4 P0,
                                        const float4 P3, Setup32& S, float4& rho, float4& c) {
  const float4 w = ray1;
  float ww = fmaf(w.x, w.x, fmaf(w.y, w.y, w.z * w.z));
  bool ok = isfinite(ray0.x) && isfinite(ray0.y) && isfinite(ray0.z) && isfinite(w.x) &&
            isfinite(w.y) && isfinite(w.z) && !(ray0.w <= 0.0f) && !isnan(ray0.w) && ww > 0.0f &&
            ww < INFINITY;
  S.iw = kUnit ? 1.0f : frsqrt(ww);
  S.lw = kUnit ? 1.0f : ww * S.iw;
  S.wh = kUnit ? w : make_float4(w.x * S.iw, w.y * S.iw, w.z * S.iw, 0.0f);
  onb(S.wh, S.b1, S.b2);
  c = make_float4(0.5f * (P0.x + P3.x), 0.5f * (P0.y + P3.y), 0.5f * (P0.z + P3.z), 0.0f);
  S.ts = fmaf(c.x - ray0.x, w.x, fmaf(c.y - ray0.y, w.y, (c.z - ray0.z) * w.z)) * frcp(ww);
  // FP64: v = c - o - ts d (exact inputs), rho = (<v,b1>, <v,b2>, <v,w^>)
  double ts = S.ts;
  double vx = fma(-ts, (double)w.x, (double)c.x - (double)ray0.x);
  double vy = fma(-ts, (double)w.y, (double)c.y - (double)ray0.y);
  double vz = fma(-ts, (double)w.z, (double)c.z - (double)ray0.z);
  rho = make_float4((float)fma(vx, (double)S.b1.x, fma(vy, (double)S.b1.y, vz * (double)S.b1.z)),
                    (float)fma(vx, (double)S.b2.x, fma(vy, (double)S.b2.y, vz * (double)S.b2.z)),
                    (float)fma(vx, (double)S.wh.x, fma(vy, (double)S.wh.y, vz * (double)S.wh.z)), 0.0f);
  return ok;
}

// ------------------------------------------------------------------------------------
// kernel parameters and record helpers
// ------------------------------------------------------------------------------------
struct Params {
  const float4* rays;
  int64_t n_rays;
  const float4 *p0, *p1, *p2, *p3;
  const uint32_t* sflags;
  int64_t n_segs;
  const uint2* pairs;
  uint32_t n_pairs;
  int depth;
  uint32_t min_size;  // 2^(23 - depth), lst:algorithm
  float4* hits;
  unsigned long long* nearest;
  int closest;  // bit 0: bound each pair's t_max by its ray's best hit so far
                // (fiber_intersect_closest); bit 1: nearest keys carry the segment index
                // instead of the pair index (fiber_grid_closest)
  unsigned int* counter;  // this call's own counters (zeroed on its stream): [0-1] K2 pair
                          // counter (64-bit), [4]/[5] list appends = list lengths for K3
  uint32_t* list_exact;   // pairs K2 flagged for the FP64 re-run   [n_pairs]
  uint32_t* list_fin;     // provisional hits for the FP64 finalise [n_pairs]
};

// Internal flags of records between the kernels (never visible after fiber_intersect
// returns): a provisional hit, and a pair to re-run in FP64; K3 consumes both.
constexpr uint32_t kProvisional = 1u << 6;
constexpr uint32_t kUncertain = 1u << 7;
constexpr uint32_t kExactLeaf = 1u << 27;  // in word y of a provisional record: FP64 leaf
constexpr int kWalk = 48;                  // K3's neighbour-leaf walk range

__device__ __forceinline__ void write_record(const Params& p, uint32_t i, uint32_t ray, float t,
                                             float u, uint32_t n_oct, uint32_t flags) {
  FIBER_CHECK(i < p.n_pairs);
  FIBER_CHECK(!(p.nearest && (flags & FIBER_HIT)) || (int64_t)ray < p.n_rays);
  if (p.hits) p.hits[i] = make_float4(t, u, __uint_as_float(n_oct), __uint_as_float(flags));
  if (p.nearest && (flags & FIBER_HIT)) {
    const uint32_t low = (p.closest & 2) ? __ldg(&p.pairs[i]).y : i;
    unsigned long long key =
        ((unsigned long long)__float_as_uint(t) << 32) | (unsigned long long)low;
    atomicMin(&p.nearest[ray], key);
  }
}

// world vector v (xyz, w = radius part) -> local frame (no translation)
__device__ __forceinline__ float4 rot(const Setup32& S, const float4 w, float4 v) {
#ifdef FIBER_PACKED
  // (<v,b1>, <v,b2>) as one packed dot product, in dot3's order of operations
  const float2 xy = __ffma2_rn(s2(v.x), make_float2(S.b1.x, S.b2.x),
                               __ffma2_rn(s2(v.y), make_float2(S.b1.y, S.b2.y),
                                          __fmul2_rn(s2(v.z), make_float2(S.b1.z, S.b2.z))));
  return make_float4(xy.x, xy.y, dot3(v, w), v.w);
#else
  return make_float4(dot3(v, S.b1), dot3(v, S.b2), dot3(v, w), v.w);
#endif
}

// ------------------------------------------------------------------------------------
// per-pair traversal state and one iteration of the loop
// ------------------------------------------------------------------------------------
struct Lane {
  Delta cur;
  float tmin, tmax, lo0, hi0, c0;
  float stmin, stmax;  // interval saved at level kCropLevel (deep backtracks)
  float delta;         // FP32 error scale of the local coordinates: 2^-20 max|coordinate|
  float terr, sterr;   // error bound of the current (saved) interval bounds
  uint32_t tie;        // 0, or after the first near-tie decision: the resume point's pending
                       // bits | the tie kinds seen (bits 0-4): re-run the pair in FP64 (K3)
  uint32_t tag, stag, bits, start, size, tests, backtracks;
  uint32_t ncache, cache_top, cache_right;  // parent-cache fill, ring top, near-side bits
};

enum : int { ST_RUNNING = 0, ST_MISS = 1, ST_HIT = 2, ST_NEED_BT = 3 };

// Per-lane shared-memory slots, component-major (stride kThreads: conflict-free): the
// ray-frame curve for re-calculation, and a ring of kFarCache parents of pending levels
// (the far child is rebuilt from its parent on backtracking, so a push is 4 plain stores).
struct HodoRef {
  float4* base;  // hodograph slot: &smem[threadIdx.x]
  float4* far;   // parent ring:    &smem[4 * kThreads + threadIdx.x]
  uint32_t* rs;  // FP64 resume point (start | log2(size) << 24), written at the first tie
  float4* wr;    // the pair's ray direction (xyz) and ray index (w bits), written at setup
  __device__ __forceinline__ void push(const Delta& f, float4 ival, uint32_t slot) const {
    FIBER_CHECK(slot < (uint32_t)kFarCache);
    float4* q = far + slot * kRingF4 * kThreads;
    q[0] = f.p;
    q[kThreads] = f.d;
    q[2 * kThreads] = f.t0;
    q[3 * kThreads] = f.t1;
    q[4 * kThreads] = ival;
  }
  __device__ __forceinline__ void pop(Delta& f, float4& ival, uint32_t slot) const {
    FIBER_CHECK(slot < (uint32_t)kFarCache);
    const float4* q = far + slot * kRingF4 * kThreads;
    f.p = q[0];
    f.d = q[kThreads];
    f.t0 = q[2 * kThreads];
    f.t1 = q[3 * kThreads];
    ival = q[4 * kThreads];
  }
  __device__ __forceinline__ void store(const Hodo& h) const {
    base[0] = h.L0;
    base[kThreads] = h.D0;
    base[2 * kThreads] = h.D1;
    base[3 * kThreads] = h.D2;
  }
  __device__ __forceinline__ Hodo load() const {
    Hodo h;
    h.L0 = base[0];
    h.D0 = base[kThreads];
    h.D1 = base[2 * kThreads];
    h.D2 = base[3 * kThreads];
    return h;
  }
};

// One prepared pair: the ray-frame curve, the ray interval and the root slab.
struct Prepared {
  Hodo h;
  float lo0, hi0, tmin, tmax, delta, terr;
  uint32_t pair, badseg, tag;
};

// a2: transform pair i's segment into its ray frame (lst:transform_curve P:1482-1512) and
// form the root interval.  Returns false for bad input (written as a miss).
__device__ __forceinline__ bool prepare(const Params& p, uint32_t i, const uint2 pr, Prepared& e,
                                        float4* wr) {
  if ((int64_t)pr.x >= p.n_rays || (int64_t)pr.y >= p.n_segs) {
    write_record(p, i, 0, INFINITY, 0.0f, 0u, FIBER_BAD_INPUT);
    return false;
  }
  const float4 ray0 = __ldg(&p.rays[2 * (int64_t)pr.x]);
  const float4 ray1 = __ldg(&p.rays[2 * (int64_t)pr.x + 1]);
  const float4 P0 = __ldg(&p.p0[pr.y]), P1 = __ldg(&p.p1[pr.y]);
  const float4 P2 = __ldg(&p.p2[pr.y]), P3 = __ldg(&p.p3[pr.y]);
  const uint32_t sf = __ldg(&p.sflags[pr.y]);
  if (kRayStash) *wr = make_float4(ray1.x, ray1.y, ray1.z, __uint_as_float(pr.x));
  e.badseg = (sf & FIBER_SEG_INVALID_MASK) != 0u ? FIBER_BAD_SEGMENT : 0u;
  e.pair = i;
  Setup32 S;
  float4 rho, c;
  if (!frame32<true>(ray0, ray1, P0, P3, S, rho, c)) {
    write_record(p, i, pr.x, INFINITY, 0.0f, 0u, FIBER_BAD_INPUT | e.badseg);
    return false;
  }
  if (!unit_dir(fmaf(ray1.x, ray1.x, fmaf(ray1.y, ray1.y, ray1.z * ray1.z)))) {
    // a non-unit direction: the whole traversal runs in FP64 (K3), from the root
    p.hits[i] = make_float4(__uint_as_float((uint32_t)FIBER_MAX_DEPTH << 24), 0.0f, 0.0f,
                            __uint_as_float(e.badseg | kUncertain));
    const uint32_t k = atomicAdd(&p.counter[4], 1u);
    FIBER_CHECK(k < p.n_pairs && i < p.n_pairs);
    p.list_exact[k] = i;
    return false;
  }
  const float4 w = S.wh;
  // differences are rotated directly, so they keep the relative precision of the inputs
  e.h.L0 = rot(S, w, P0 - c) + rho;
  e.h.L0.w = P0.w;
  if (sf & FIBER_SEG_QUADRATIC) {
    // exact degree elevation of (q0, q1, q2) = (P0, P1, P3) from the rotated differences:
    // Q1 - Q0 = 2/3 (q1 - q0), Q2 - Q1 = 1/3 (q2 - q0), Q3 - Q2 = 2/3 (q2 - q1)
    const float4 a = rot(S, w, P1 - P0), b = rot(S, w, P3 - P1);
    e.h.D0 = 0.6666666865348816f * a;
    e.h.D1 = 0.3333333432674408f * (a + b);
    e.h.D2 = 0.6666666865348816f * b;
  } else {
    e.h.D0 = rot(S, w, P1 - P0);
    e.h.D1 = rot(S, w, P2 - P1);
    e.h.D2 = rot(S, w, P3 - P2);
  }
  // ray interval [0, tmax) in local z units: z = (t - ts) |d|
  e.lo0 = -S.ts * S.lw;
  float tlim = ray0.w;
  if (p.closest & 1) {
    // the ray's t_max as a running bound: the best hit of the
    // ray so far (read from L2, where the atomicMin of write_record lands), widened by
    // 2^-19 relative so that hits within FP32 rounding of it still compete for the minimum
    const unsigned long long key = __ldcg(&p.nearest[pr.x]);
    if (key != ~0ull) {
      const float tb = __uint_as_float((uint32_t)(key >> 32));
      tlim = fminf(tlim, fmaf(tb, 1.9073486328125e-06f, tb) + 1e-30f);
    }
  }
  e.hi0 = (tlim - S.ts) * S.lw;
  Delta cur;  // conversion {p0,p1,p2,p3} -> {p,d,t0,t1} (3.1 P:372-375)
  cur.p = e.h.L0;
  cur.d = e.h.D0 + e.h.D1 + e.h.D2;
  cur.t0 = e.h.D0;
  cur.t1 = e.h.D2;
  float kappa;
  slab(cur, e.lo0, e.hi0, 0u, 1u << FIBER_MAX_DEPTH, e.tmin, e.tmax, e.tag, false, &kappa);
  // FP32 error scale: 2^-20 of the largest local coordinate of the control points
  const float4 L1 = e.h.L0 + e.h.D0, L3 = e.h.L0 + cur.d, L2 = L3 - e.h.D2;
  auto amax = [](float4 v) { return fmaxf(fabsf(v.x), fmaxf(fabsf(v.y), fabsf(v.z))); };
  e.delta = 9.5367431640625e-07f * fmaxf(fmaxf(amax(e.h.L0), amax(L1)), fmaxf(amax(L2), amax(L3)));
  e.terr = e.delta * (1.0f + kappa);
  return true;
}

// Record near-tie kinds t of the current node's decisions.  At the first one, the FP64
// re-run's resume point is fixed: every earlier decision was certain, so the FP64 traversal
// may start at this node (its curve and interval re-derived exactly) with the pending
// levels above it.  Below the crop level the FP32 path is uncropped and may have strayed
// from the oracle's, so the resume point is the node's crop-level ancestor (the pending bits
// of deeper levels dropped).  Pending far children above the resume node are at least
// kCropMinSize, so bits 0-4 are free for the kinds.
__device__ __forceinline__ void note_tie(Lane& L, HodoRef hs, uint32_t t) {
  if (t != 0u && L.tie == 0u) {
    const bool deep = L.size < kCropMinSize;
    const uint32_t st = deep ? (L.start & ~(kCropMinSize - 1u)) : L.start;
    const uint32_t sz = deep ? kCropMinSize : L.size;
    *hs.rs = st | ((31u - __clz(sz)) << 24);
    L.tie = deep ? (L.bits & ~(kCropMinSize - 1u)) : L.bits;
  }
  L.tie |= t;
}

// One iteration: node test, then descend.  Returns ST_RUNNING, ST_MISS, ST_HIT (leaf
// accepted; L.c0 holds the cylinder entry) or ST_NEED_BT (pruned with levels pending).
__device__ __forceinline__ int step(Lane& L, HodoRef hs, uint32_t min_size) {
  ++L.tests;
  float c0, c1, tie_e, inv_sin;
  const bool cyl = cylinder(L.cur, c0, c1, &tie_e, &inv_sin, L.delta);
  // pruning test P:1618 with F1 (empty interval) and F5 (explicit miss)
  bool pass = cyl && (c1 >= L.tmin) && (c0 <= L.tmax) && (L.tmin <= L.tmax);
  // near-ties of the test (R5): the entry/exit parameters carry an error of about
  // delta / sin(ray, axis), the interval bounds L.terr
  const float tau = L.delta * fmaf(2.0f, inv_sin, 2.0f);
  const float tb = tau + L.terr;
  note_tie(L, hs, (tie_e < 0.0f ? 1u : 0u) |
                  ((cyl && ((fabsf(c1 - L.tmin) < tb) | (fabsf(L.tmax - c0) < tb) |
                            (fabsf(L.tmax - L.tmin) < 2.0f * L.terr))) ? 2u : 0u));
  // a5 for a cached far child is folded into the descent below: jump_up to the deepest
  // pending level (the most recent push), then the far child of the cached parent is built
  // with the same split arithmetic as the near child was, and its interval is the parent's
  // with the split plane as its lower bound (a pending far child has c0 < t_P < c1, so the
  // near child ended at t_P) -- its own slab (F7) in exact arithmetic.
  bool bt = false, near_right = false;
  if (!pass) {
    if (L.bits == 0u) return ST_MISS;        // done
    if (L.ncache == 0u) return ST_NEED_BT;   // re-calculation path (backtrack())
    bt = true;
    ++L.backtracks;
    L.size = L.bits & (0u - L.bits);  // lowest pending bit (ctz), lst:bitstring P:1530-1542
    L.start ^= L.size;
    L.bits ^= L.size;
    L.start &= ~(L.size - 1u);
    float4 iv;
    hs.pop(L.cur, iv, L.cache_top);  // the parent
    near_right = (L.cache_right >> L.cache_top) & 1u;
    L.cache_top = (L.cache_top + kFarCache - 1u) % kFarCache;
    --L.ncache;
    L.tmin = iv.x;
    L.tmax = iv.y;
    L.tag = __float_as_uint(iv.z);
    L.terr = iv.w;
  } else if (L.size <= min_size) {  // leaf: first hit terminates
    // the kind decision (F2, F6) matters only where the bound is a global cap or the ray
    // origin: LATERAL and WEDGE are one class with the same values (R3)
    const bool cap_bound = L.tag == TAG_ORIGIN || (L.tag == 0u && L.start == 0u) ||
                           (L.tag == (1u << FIBER_MAX_DEPTH) &&
                            L.start + L.size == (1u << FIBER_MAX_DEPTH));
    note_tie(L, hs, (cap_bound && fabsf(c0 - L.tmin) < tb) ? 4u : 0u);
    // below the crop level the leaf index is only known to about (error of c0 along the
    // axis) / (leaf length) = tau |d_z| / |d|^2 leaves; K3 walks up to kWalk of them, so
    // nearly parallel rays that could be further off are re-run in FP64
    // An INSIDE entry (the origin bounds t_min) below the crop level is re-run too: the FP32
    // descent there orders children by the cylinder entry behind the origin and does not crop,
    // so its leaf can be far from the one holding the origin.
    if (L.size < kCropMinSize)
      note_tie(L, hs, (L.delta * inv_sin * fabsf(L.cur.d.z) > (float)kWalk * dot3(L.cur.d, L.cur.d) ||
                       (L.tag == TAG_ORIGIN && !(c0 >= L.tmin))) ? 8u : 0u);
    L.c0 = c0;
    return ST_HIT;
  }
  // the node being split (the current node, or the cached parent) and its plane
  // (lst:subdivide_partition_and_update P:1429-1456)
  const uint32_t psize = bt ? 2u * L.size : L.size;
  const bool crop = psize > kCropMinSize;
  Split sp;
  split_geometry(L.cur, sp);
  const float num = dot3(sp.tcn, sp.S), nz = sp.tcn.z;
  const float rz = frcp(nz);
  const float tP = num * rz;
  const float kP = fminf((fabsf(sp.tcn.x) + fabsf(sp.tcn.y) + fabsf(nz)) * fabsf(rz), 1e30f);
  const bool par = (nz == 0.0f);
  const float tauP = L.delta * (1.0f + kP);
  bool right;
  if (!bt) {
    right = par ? (num < 0.0f) : ((tP > c0) != (nz > 0.0f));  // near child (F9)
    const bool both = !par && (c0 < tP) && (tP < c1);
    const float4 ival = make_float4(L.tmin, L.tmax, __uint_as_float(L.tag), L.terr);
    // one-bound update down to the crop level
    const bool apply = crop && !par, up = tP > c0;
    const bool hi_up = apply && up && tP < L.tmax;
    const bool lo_up = apply && !up && tP > L.tmin;
    L.tmax = hi_up ? tP : L.tmax;
    L.tmin = lo_up ? tP : L.tmin;
    L.tag = lo_up ? L.start + (L.size >> 1) : L.tag;
    if (crop) {
      // near-ties of the near-child / both decisions and the error of the updated bound.
      // Below the crop level these decisions only pick among nearly collinear leaves, so
      // they are not re-run.
      note_tie(L, hs, ((fabsf(tP - c0) < tau + tauP) | (fabsf(tP - c1) < tau + tauP)) ? 16u : 0u);
      if (hi_up | lo_up) L.terr = fmaxf(L.terr, tauP);
    }
    // go_down (lst:bitstring_manipulation P:1516-1528)
    L.size >>= 1;
    if (both) {
      // remember the parent and its interval: the next jump_up returns to the deepest
      // pending level, i.e. the most recent push (LIFO); the ring drops the oldest entry
      L.bits |= L.size;
      L.cache_top = (L.cache_top + 1u) % kFarCache;
      hs.push(L.cur, ival, L.cache_top);
      L.cache_right = right ? (L.cache_right | (1u << L.cache_top))
                               : (L.cache_right & ~(1u << L.cache_top));
      L.ncache = min(L.ncache + 1u, (uint32_t)kFarCache);
    }
    if (right) L.start |= L.size;
  } else {
    right = !near_right;
    // the far child starts at the split plane (its tag: the split's u)
    const bool lo_up = crop && tP > L.tmin;
    L.tmin = lo_up ? tP : L.tmin;
    L.tag = lo_up ? (right ? L.start : L.start + L.size) : L.tag;
    if (lo_up) L.terr = fmaxf(L.terr, tauP);
  }
  child(L.cur, sp, right, L.cur);
  if (L.size == kCropMinSize) {
    L.stmin = L.tmin;
    L.stmax = L.tmax;
    L.stag = L.tag;
    L.sterr = L.terr;
  }
  return ST_RUNNING;
}

// jump_up to the deepest pending level when its parent is not in the ring:
// the far node's curve re-calculated and its own interval (F7).
__device__ __forceinline__ void backtrack(Lane& L, HodoRef hs) {
  ++L.backtracks;
  L.size = L.bits & (0u - L.bits);  // lowest pending bit (ctz)
  L.start ^= L.size;
  L.bits ^= L.size;
  L.start &= ~(L.size - 1u);
  constexpr bool cached = false;  // cached far children are built inside step()
  {
    float u0, u1;
    get_interval(L.start, L.size, u0, u1);
    recompute(hs.load(), u0, u1, L.cur);  // lst:recalculation P:1371-1385
  }
  if (L.size >= kCropMinSize) {
    float kappa;
    slab(L.cur, L.lo0, L.hi0, L.start, L.start + L.size, L.tmin, L.tmax, L.tag, !cached, &kappa);
    L.terr = L.delta * (1.0f + kappa) * (cached ? 1.0f : 4.0f);
    if (L.size == kCropMinSize) {
      L.stmin = L.tmin;
      L.stmax = L.tmax;
      L.stag = L.tag;
      L.sterr = L.terr;
    }
  } else {
    L.tmin = L.stmin;
    L.tmax = L.stmax;
    L.tag = L.stag;
    L.terr = L.sterr;
  }
}

__device__ __forceinline__ void list_append(uint32_t* list, uint32_t k, uint32_t i, const Params& p) {
  FIBER_CHECK(k < p.n_pairs && i < p.n_pairs);
  list[k] = i;
}

__device__ __forceinline__ uint32_t counter_bits(const Lane& L) {
  return (min(L.backtracks, 255u) << 8) | (min(L.tests, 65535u) << 16);
}

// Pair ended with status st: write the miss, or the provisional hit record for K3
// (z* bits, start | kind << 24 | inside << 26, tag of t_min, counters | bad_segment |
// kProvisional).
#ifndef FIBER_FP32_FIN_DEPTH
#define FIBER_FP32_FIN_DEPTH FIBER_MAX_DEPTH
#endif
__device__ __forceinline__ void end_pair(const Params& p, uint32_t i, const Lane& L, int st,
                                         uint32_t badseg, HodoRef hs) {
  if (L.tie) {  // decided by a near-tie somewhere: K3 re-runs the pair in FP64
    p.hits[i] = make_float4(__uint_as_float(*hs.rs), __uint_as_float(L.tie & 31u),
                            __uint_as_float(L.tie & ~31u), __uint_as_float(badseg | kUncertain));
    list_append(p.list_exact, atomicAdd(&p.counter[4], 1u), i, p);
    return;
  }
  if (st == ST_HIT) {
    // F2: entry into the cropped cylinder; F6: kind from the binding constraint
    const float zs = fmaxf(L.c0, L.tmin);
    uint32_t kind = FIBER_KIND_LATERAL, inside = 0;
    if (!(L.c0 >= L.tmin)) {
      if (L.tag == TAG_ORIGIN) inside = 1, kind = FIBER_KIND_WEDGE;
      else if (L.tag == 0u && L.start == 0u) kind = FIBER_KIND_CAP0;
      else if (L.tag == (1u << FIBER_MAX_DEPTH) && L.start + L.size == (1u << FIBER_MAX_DEPTH))
        kind = FIBER_KIND_CAP1;
      else kind = FIBER_KIND_WEDGE;
    }
    if (zs < L.hi0) {  // strictly before the RAY's t_max
      // a7 in FP32 when that is accurate enough: the leaf is exact (down to the crop level)
      // and the FP32 coordinate error is far below the radius (normal error ~ delta / r);
      // otherwise a provisional record for K3's FP64 re-solve
      if (!inside && p.depth <= FIBER_FP32_FIN_DEPTH && L.delta < 1.220703125e-4f * L.cur.p.w) {
        const float4 w = *hs.wr;  // stashed at setup: no dependent pair -> ray reload
        const uint2 pr = make_uint2(__float_as_uint(w.w), 0u);
        const float4 wh = w;  // a unit direction (prepare), as frame32<true>
        float4 b1, b2;
        onb(wh, b1, b2);
        const float t = zs - L.lo0;  // (z - lo0) / |d|, |d| = 1
        float u, nx, ny, nz;
        if (kind == FIBER_KIND_CAP0 || kind == FIBER_KIND_CAP1) {
          const Hodo h = hs.load();
          const float4 tg = kind == FIBER_KIND_CAP0 ? (-1.0f) * h.D0 : h.D2;
          u = kind == FIBER_KIND_CAP0 ? 0.0f : 1.0f;
          nx = tg.x;
          ny = tg.y;
          nz = tg.z;
        } else {  // u by projection onto the leaf chord, normal from the axis point
          const Delta& c = L.cur;
          float ul = fmaf(-c.p.x, c.d.x, fmaf(-c.p.y, c.d.y, (zs - c.p.z) * c.d.z)) *
                     frcp(dot3(c.d, c.d));
          // clamped to the leaf down to the crop level, where the leaf is the
          // oracle's; below it the FP32 leaf may be a few leaves off (bounded by the leaf-index
          // tie), so the clamp is to the segment: the leaf chord's extension stays within
          // curvature x offset^2 of the curve, where a leaf clamp would tilt the normal by
          // offset x leaf length / r
          if (L.size >= kCropMinSize) {
            ul = fminf(1.0f, fmaxf(0.0f, ul));
          } else {
            const float isz = frcp((float)L.size);
            ul = fminf((float)((1u << FIBER_MAX_DEPTH) - L.start) * isz, fmaxf(-(float)L.start * isz, ul));
          }
          u = fminf(1.0f, fmaxf(0.0f, fmaf(ul, (float)L.size, (float)L.start) * 1.1920928955078125e-07f));  // 2^-23
          nx = -fmaf(ul, c.d.x, c.p.x);
          ny = -fmaf(ul, c.d.y, c.p.y);
          nz = zs - fmaf(ul, c.d.z, c.p.z);
        }
        // back to world coordinates
        const float wx = fmaf(nx, b1.x, fmaf(ny, b2.x, nz * wh.x));
        const float wy = fmaf(nx, b1.y, fmaf(ny, b2.y, nz * wh.y));
        const float wz = fmaf(nx, b1.z, fmaf(ny, b2.z, nz * wh.z));
        write_record(p, i, pr.x, t, u, encode_oct_f(wx, wy, wz),
                     FIBER_HIT | (kind << FIBER_KIND_SHIFT) | counter_bits(L) | badseg);
        return;
      }
      p.hits[i] = make_float4(zs, __uint_as_float(L.start | (kind << 24) | (inside << 26)),
                              __uint_as_float(L.tag),
                              __uint_as_float(counter_bits(L) | badseg | kProvisional));
      list_append(p.list_fin, atomicAdd(&p.counter[5], 1u), i, p);
      return;
    }
  }
  p.hits[i] = make_float4(INFINITY, 0.0f, 0.0f, __uint_as_float(badseg | counter_bits(L)));
}

// a7 for one provisional hit (all lanes of the batch run it together, converged).
__device__ __noinline__ void finalize_one(const Params& p, uint32_t i) {
  FIBER_CHECK(i < p.n_pairs);
  const float4 rec = p.hits[i];
  const uint2 pr = __ldg(&p.pairs[i]);
  FIBER_CHECK((int64_t)pr.x < p.n_rays && (int64_t)pr.y < p.n_segs);
  const float4 ray0 = __ldg(&p.rays[2 * (int64_t)pr.x]);
  const float4 ray1 = __ldg(&p.rays[2 * (int64_t)pr.x + 1]);
  const float4 P0 = __ldg(&p.p0[pr.y]), P1 = __ldg(&p.p1[pr.y]);
  const float4 P2 = __ldg(&p.p2[pr.y]), P3 = __ldg(&p.p3[pr.y]);
  const uint32_t y = __float_as_uint(rec.y);
  uint32_t start = y & 0x00ffffffu, kind = (y >> 24) & 3u;
  bool inside = (y >> 26) & 1u;
  const bool exact_leaf = (y & kExactLeaf) != 0u;
  const uint32_t lo_tag = __float_as_uint(rec.z);
  uint32_t flags = __float_as_uint(rec.w) & ~kProvisional;
  // the FP32 z* as a ray parameter (only used for WEDGE entries); an INSIDE entry is the ray
  // origin itself, t* = 0 (F2 with t_min = 0; a re-run record carries no z*)
  Setup32 S;
  float4 rho, c;
  frame32<false>(ray0, ray1, P0, P3, S, rho, c);
  float t32 = inside ? 0.0f : fmaf(rec.x, S.iw, S.ts);
  float t, u;
  uint32_t n_oct;
  bool hit;
  // the FP32 leaf is exact down to the crop level; below it (and not re-run in FP64) it is
  // searched for within kWalk leaves
  const int walk = (exact_leaf || p.depth <= kCropLevel) ? 0 : kWalk;
  const bool quad = (__ldg(&p.sflags[pr.y]) & FIBER_SEG_QUADRATIC) != 0u;
  finalize(ray0, ray1, P0, P1, P2, P3, quad, start, p.depth, kind, lo_tag, t32, walk, t, u, n_oct, hit,
           kind);
  if (inside && hit) {
    t = 0.0f;
    kind = FIBER_KIND_LATERAL;
  }
  if (hit) flags |= FIBER_HIT | (kind << FIBER_KIND_SHIFT) | (inside ? FIBER_INSIDE : 0u);
  write_record(p, i, pr.x, t, u, n_oct, flags);
}

// ------------------------------------------------------------------------------------
// K2, the traversal kernel: persistent warps whose lanes are refilled in epochs
// (DESIGN.md "Kernel").  Every kEpoch iterations the warp votes; once at least kRefill
// lanes are idle they all take new pairs from one atomicAdd and run setup together, so
// setup and the loop both execute with most lanes active.  A pair runs from setup to its
// end in one lane without interruption, so its result is a deterministic function of the
// pair alone (independent of the launch shape and of the schedule).  Hits leave
// provisional records that K3 finalises.
// ------------------------------------------------------------------------------------
#ifndef FIBER_EPOCH
#define FIBER_EPOCH 2
#endif
#ifndef FIBER_REFILL
#define FIBER_REFILL 16
#endif
constexpr int kEpoch = FIBER_EPOCH;          // iterations between refill votes
constexpr uint32_t kRefill = FIBER_REFILL;  // idle lanes that trigger a refill

__device__ __forceinline__ void start_lane(const Prepared& e, Lane& L, HodoRef hs) {
  hs.store(e.h);
  L.cur.p = e.h.L0;
  L.cur.d = e.h.D0 + e.h.D1 + e.h.D2;
  L.cur.t0 = e.h.D0;
  L.cur.t1 = e.h.D2;
  L.lo0 = e.lo0;
  L.hi0 = e.hi0;
  L.tmin = L.stmin = e.tmin;
  L.tmax = L.stmax = e.tmax;
  L.tag = L.stag = e.tag;
  L.delta = e.delta;
  L.terr = L.sterr = e.terr;
  L.tie = 0u;
  L.bits = 0;
  L.size = 1u << FIBER_MAX_DEPTH;
  L.start = 0;
  L.tests = 0;
  L.backtracks = 0;
  L.c0 = 0.0f;
  L.ncache = 0;
  L.cache_top = 0;
  L.cache_right = 0;
}

#ifndef FIBER_K2_MINBLOCKS
#define FIBER_K2_MINBLOCKS 3
#endif
__global__ void __launch_bounds__(kThreads, FIBER_K2_MINBLOCKS) intersect_kernel(const Params p) {
  extern __shared__ float4 smem[];
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t lt = (1u << lane) - 1u;
  HodoRef hs{&smem[threadIdx.x], &smem[4 * kThreads + threadIdx.x],
             reinterpret_cast<uint32_t*>(&smem[(4 + kRingF4 * kFarCache) * kThreads]) + threadIdx.x,
             &smem[(4 + kRingF4 * kFarCache) * kThreads + kThreads / 4 + threadIdx.x]};
  const uint32_t min_size = p.min_size;
  Lane L;
  uint32_t pair = 0, badseg = 0;
  int ended = ST_RUNNING;  // a finished pair whose record is not written yet
  bool active = false, drained = false;
  // The pair counter is 64-bit (slot words 0-1): claims past n_pairs cannot wrap.
  unsigned long long* const pair_counter = reinterpret_cast<unsigned long long*>(p.counter);
  while (true) {
    const unsigned idle = __ballot_sync(0xffffffffu, !active);
    if (!drained && (__popc(idle) >= (int)kRefill || idle == 0xffffffffu)) {
      // the claim first: its atomic's latency overlaps the record writing below
      const uint32_t k = __popc(idle), r = __popc(idle & lt);
      unsigned long long claimed = 0;
      if (lane == 0) claimed = atomicAdd(pair_counter, (unsigned long long)k);
      // a6-a7 for the lanes that finished since the last refill, together (the lane keeps
      // its state until then), so the record writer runs at the refill's SIMT width
      if (ended != ST_RUNNING) {
        end_pair(p, pair, L, ended, badseg, hs);
        ended = ST_RUNNING;
      }
      uint32_t base = (uint32_t)min(claimed, (unsigned long long)p.n_pairs);
      base = __shfl_sync(0xffffffffu, base, 0);
      if (base + k >= p.n_pairs) {
        drained = true;
      }
      if (!active) {
        const uint32_t i = base + r;
        FIBER_CHECK(base <= p.n_pairs);
        if (i < p.n_pairs) {
          const uint2 pr = __ldg(&p.pairs[i]);
          Prepared e;
          if (prepare(p, i, pr, e, hs.wr)) {  // a2
            start_lane(e, L, hs);
            pair = e.pair;
            badseg = e.badseg;
            active = true;
          }
        }
      }
    }
    if (__ballot_sync(0xffffffffu, active) == 0u) {
      if (drained) break;
      continue;
    }
#pragma unroll 1
    for (int k = 0; k < kEpoch; ++k) {
      if (active) {
        const int st = step(L, hs, min_size);  // a3-a4
        if (st == ST_NEED_BT) backtrack(L, hs);  // a5
        // a pair ends at its leaf or miss -- or at its first near-tie decision: K3 re-runs
        // it in FP64 from that node on, so the rest of its FP32 traversal would be discarded
        if ((st != ST_RUNNING && st != ST_NEED_BT) || L.tie != 0u) {
          ended = st == ST_HIT ? ST_HIT : ST_MISS;  // a6-a7 at the next refill (or the exit)
          active = false;
        }
      }
    }
  }
  if (ended != ST_RUNNING) end_pair(p, pair, L, ended, badseg, hs);
  // this warp has no pairs left: K3 (a programmatic dependent) may be scheduled once every
  // block got here; it still waits for K2's completion before reading anything
  asm volatile("griddepcontrol.launch_dependents;");
}

// ------------------------------------------------------------------------------------
// The FP64 re-run of a pair K2 flagged as decided by a near-tie (R5): the whole
// traversal in double precision (exact.cuh), leaving a provisional record (with its exact
// leaf) or the final miss.  Runs inside K3, queued with the provisional hits.
// ------------------------------------------------------------------------------------
__device__ __noinline__ void exact_one(const Params& p, uint32_t i) {
  const uint32_t badseg = __float_as_uint(p.hits[i].w) & FIBER_BAD_SEGMENT;
  const uint2 pr = __ldg(&p.pairs[i]);
  const float4 ray0 = __ldg(&p.rays[2 * (int64_t)pr.x]);
  const float4 ray1 = __ldg(&p.rays[2 * (int64_t)pr.x + 1]);
  const float4 P0 = __ldg(&p.p0[pr.y]), P1 = __ldg(&p.p1[pr.y]);
  const float4 P2 = __ldg(&p.p2[pr.y]), P3 = __ldg(&p.p3[pr.y]);
  const bool quad = (__ldg(&p.sflags[pr.y]) & FIBER_SEG_QUADRATIC) != 0u;
  // resume where K2 saw its first near-tie (note_tie): start | log2(size) << 24, bits
  const float4 rec = p.hits[i];
  const uint32_t rs = __float_as_uint(rec.x), rbits = __float_as_uint(rec.z);
  const uint32_t rstart = rs & 0x00ffffffu, rsize = 1u << (rs >> 24);
  const exact::Result r = exact::traverse(ray0, ray1, P0, P1, P2, P3, quad, p.depth, rstart,
                                          rsize, rbits);
  const uint32_t cnt = (min(r.backtracks, 255u) << 8) | (min(r.tests, 65535u) << 16);
  if (r.hit) {
    p.hits[i] = make_float4(0.0f, __uint_as_float(r.start | (r.kind << 24) | (r.inside << 26) | kExactLeaf),
                            __uint_as_float(r.tag), __uint_as_float(cnt | badseg | kProvisional));
  } else {
    p.hits[i] = make_float4(INFINITY, 0.0f, 0.0f, __uint_as_float(cnt | badseg));
  }
}

// ------------------------------------------------------------------------------------
// K3, the finalisation kernel: scans the records, queues provisional hits per warp and
// finalises them in FP64 32 at a time (converged).  a7, lst:calc_intersection P:1546-1587.
// ------------------------------------------------------------------------------------
// K3: 128-thread blocks, 3 per SM = 12 warps/SM at <= 170 registers (the FP64 path must not
// spill: a cold local-memory reload on a latency-bound chain costs more than occupancy).
constexpr int kK3Threads = 128;
#ifndef FIBER_K3_MINBLOCKS
#define FIBER_K3_MINBLOCKS 3
#endif
__global__ void __launch_bounds__(kK3Threads, FIBER_K3_MINBLOCKS) finalize_kernel(const Params p) {
  // K3 walks the two lists K2 appended to.  The FP64 re-runs are long dependent chains
  // (latency-, not throughput-bound), so they are dealt round-robin over ALL warps of the
  // grid first -- item k to warp k mod W, lane k / W -- and a short list runs one lane per
  // warp with no divergence; a re-run that hits is finalised by the same lane.  No atomics:
  // both lists are dealt statically from the lengths K2's last block published.
  const uint32_t lane = threadIdx.x & 31u;
  // launched as a programmatic dependent of K2 (launch_intersect): wait until K2 has
  // completed and its memory (records, lists, list lengths) is visible
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t n_exact = p.counter[4];
  const uint32_t n_fin = p.counter[5];
  const uint32_t W = gridDim.x * (blockDim.x >> 5);
  const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
#ifndef FIBER_NO_EXACT
  // 32-bit indices (64-bit ones made this loop 3x slower on C4): n_pairs < 2^31 (fiber.h) and
  // W * 32 < 2^17, so k never wraps
  for (uint32_t k = gw + W * lane; k < n_exact; k += W * 32u) {
    FIBER_CHECK(k < p.n_pairs);
    const uint32_t i = p.list_exact[k];
    FIBER_CHECK(i < p.n_pairs);
    exact_one(p, i);  // the FP64 traversal, then the finalisation if it hit
    if (__float_as_uint(p.hits[i].w) & kProvisional) finalize_one(p, i);
  }
#endif
#ifndef FIBER_NO_FIN
  // 32 provisional hits per warp, chunks dealt from the last warp down so the warps that
  // hold re-runs get them last
  for (uint32_t c = W - 1u - gw; c * 32u < n_fin; c += W)
    if (c * 32u + lane < n_fin) {
      FIBER_CHECK(c * 32u + lane < p.n_pairs && p.list_fin[c * 32u + lane] < p.n_pairs);
      finalize_one(p, p.list_fin[c * 32u + lane]);
    }
#endif
}

// K4, the per-ray nearest keys of fiber_intersect_nearest (no running bound): one pass over
// the finished records, atomicMin((bits(t) << 32) | i) into nearest[ray] for every hit --
// the same keys write_record would have formed.  Run after K3 instead of inside K2 because
// K2's reductions there share the L2 atomic units with its pair-claim atomics and stall the
// refills (C5 2.06 -> 3.02 ms per 2^25-pair chunk with them inline).
__global__ void __launch_bounds__(256) nearest_kernel(const Params p, unsigned long long* nearest) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < p.n_pairs;
       i += gridDim.x * blockDim.x) {
    const float4 r = __ldcs(&p.hits[i]);
    if (__float_as_uint(r.w) & FIBER_HIT) {
      const uint32_t ray = __ldg(&p.pairs[i]).x;
      FIBER_CHECK((int64_t)ray < p.n_rays);
      atomicMin(&nearest[ray], ((unsigned long long)__float_as_uint(r.x) << 32) | i);
    }
  }
}

__global__ void fill_u64(unsigned long long* p, int64_t n, unsigned long long v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

}  // namespace fiberx

using namespace fiberx;

// Per-device launch constants, queried once per process and device (immutable afterwards;
// a call otherwise spends far longer in these queries than the GPU spends on 1M pairs).
struct LaunchInfo {
  int sms, k2_per_sm, k3_per_sm;
};
constexpr size_t kCounterBytes = 256;  // per-call work counters at the head of the scratch

static const LaunchInfo* launch_info() {
  static std::mutex mu;
  static LaunchInfo info[64];
  static bool ready[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!ready[dev]) {
    LaunchInfo li{};
    cudaDeviceGetAttribute(&li.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(intersect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kSmemBytes);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&li.k2_per_sm, intersect_kernel, kThreads,
                                                  kSmemBytes);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&li.k3_per_sm, finalize_kernel, kK3Threads, 0);

    if (li.k2_per_sm < 1) li.k2_per_sm = 1;
    if (li.k3_per_sm < 1) li.k3_per_sm = 1;
    if (cudaGetLastError() != cudaSuccess || li.sms < 1) return nullptr;
    info[dev] = li;
    ready[dev] = true;
  }
  return &info[dev];
}


// The per-call scratch (two work lists of n_pairs entries, and records when the caller
// gives none) comes from a private stream-ordered memory pool per device that keeps its
// memory (no system calls after warm-up, no effect on the application's default pool).
cudaMemPool_t scratch_pool(int dev) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  std::lock_guard<std::mutex> lock(mu);
  if (!pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if (cudaMemPoolCreate(&pools[dev], &props) != cudaSuccess) return nullptr;
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
  }
  return pools[dev];
}

static int launch_intersect(const fiber_ray* rays, int64_t n_rays, const fiber_segments* segs,
                            const fiber_pair* pairs, int64_t n_pairs, int max_depth,
                            fiber_hit* hits, uint64_t* nearest, void* event_after_traverse,
                            void* stream, int closest = 0) {
  if (n_rays < 0 || n_pairs < 0 || n_rays >= ((int64_t)1 << 32) ||
      n_pairs >= ((int64_t)1 << 31) || max_depth < 0 || max_depth > FIBER_MAX_DEPTH || !segs)
    return set_error(FIBER_EINVAL, "fiber_intersect: bad size or depth");
  if (n_pairs > 0 && (!rays || !pairs || (!hits && !nearest) || !segs->p0 || !segs->p1 ||
                      !segs->p2 || !segs->p3 || !segs->flags))
    return set_error(FIBER_EINVAL, "fiber_intersect: NULL pointer");
  int rc = check_device();
  if (rc != FIBER_OK) return rc;
  if (n_pairs == 0) return FIBER_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const LaunchInfo* li = launch_info();
  if (!li) return set_error(FIBER_ECUDA, "fiber_intersect: device query failed");
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool = scratch_pool(dev);
  // the call's counters, the lists, the records (16-B float4 stores) at 256-B boundaries;
  // every call owns its counters, so any number of calls may be in flight on any streams
  const size_t list_bytes =
      kCounterBytes + ((2 * (size_t)n_pairs * sizeof(uint32_t) + 255) & ~(size_t)255);
  const size_t rec_bytes = hits ? 0 : (size_t)n_pairs * sizeof(fiber_hit);
  void* scratch = nullptr;
  cudaError_t e = pool ? cudaMallocFromPoolAsync(&scratch, list_bytes + rec_bytes, pool, st)
                       : cudaErrorMemoryAllocation;
  if (e != cudaSuccess) {
    char buf[300];
    snprintf(buf, sizeof(buf), "fiber_intersect: scratch: %s", cudaGetErrorString(e));
    return set_error(FIBER_ECUDA, buf);
  }
  if (!hits) hits = (fiber_hit*)((char*)scratch + list_bytes);
  unsigned int* counter = (unsigned int*)scratch;
  e = cudaMemsetAsync(counter, 0, 32, st);
  if (e != cudaSuccess) {
    cudaFreeAsync(scratch, st);
    return set_error(FIBER_ECUDA, "fiber_intersect: counter memset failed");
  }
  Params p;
  p.rays = (const float4*)rays;
  p.n_rays = n_rays;
  p.p0 = (const float4*)segs->p0;
  p.p1 = (const float4*)segs->p1;
  p.p2 = (const float4*)segs->p2;
  p.p3 = (const float4*)segs->p3;
  p.sflags = segs->flags;
  p.n_segs = segs->n;
  p.pairs = (const uint2*)pairs;
  p.n_pairs = (uint32_t)n_pairs;
  p.depth = max_depth;
  p.min_size = 1u << (FIBER_MAX_DEPTH - max_depth);
  p.hits = (float4*)hits;
  // fiber_intersect_nearest: the keys are formed by K4 after K3 (nearest_kernel), so K2 and
  // K3 run as for fiber_intersect; with a running bound (closest) they need them at once
#ifdef FIBER_NEAREST_INLINE  // test build: the keys inside K2/K3
  const bool defer = false;
#else
  const bool defer = nearest && closest == 0;
#endif
  p.nearest = defer ? nullptr : (unsigned long long*)nearest;
  p.closest = closest;
  p.counter = counter;
  p.list_exact = (uint32_t*)((char*)scratch + kCounterBytes);
  p.list_fin = p.list_exact + n_pairs;
  int64_t chunks = (n_pairs + 31) / 32;
  int64_t blocks = (int64_t)li->sms * li->k2_per_sm;
  if (blocks * kWarps > chunks) blocks = (chunks + kWarps - 1) / kWarps;
  intersect_kernel<<<(unsigned)blocks, kThreads, kSmemBytes, st>>>(p);
  rc = check_launch("fiber_intersect (traverse)");
  if (rc == FIBER_OK && event_after_traverse) cudaEventRecord((cudaEvent_t)event_after_traverse, st);
  if (rc == FIBER_OK) {
    const int64_t fblocks = (int64_t)li->sms * li->k3_per_sm;
    // Programmatic dependent launch: K3's launch is processed while K2 drains, and K3 waits
    // for K2's completion on the device (griddepcontrol.wait) -- not with an event in between
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)fblocks);
    cfg.blockDim = dim3(kK3Threads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
#ifdef FIBER_NO_PDL  // test build: plain stream order
    attr[0].val.programmaticStreamSerializationAllowed = 0;
#else
    attr[0].val.programmaticStreamSerializationAllowed = event_after_traverse ? 0 : 1;
#endif
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, finalize_kernel, p);
    rc = check_launch("fiber_intersect (finalize)");
  }
  if (rc == FIBER_OK && defer) {
    int64_t nblocks = (n_pairs + 255) / 256;
    if (nblocks > (int64_t)li->sms * 8) nblocks = (int64_t)li->sms * 8;
    nearest_kernel<<<(unsigned)nblocks, 256, 0, st>>>(p, (unsigned long long*)nearest);
    rc = check_launch("fiber_intersect (nearest)");
  }
  cudaFreeAsync(scratch, st);
  return rc;
}

extern "C" int fiber_intersect(const fiber_ray* rays, int64_t n_rays, const fiber_segments* segs,
                               const fiber_pair* pairs, int64_t n_pairs, int max_depth,
                               fiber_hit* hits, void* cuda_stream) {
  if (n_pairs > 0 && !hits) return set_error(FIBER_EINVAL, "fiber_intersect: NULL hits");
  return launch_intersect(rays, n_rays, segs, pairs, n_pairs, max_depth, hits, nullptr, nullptr,
                          cuda_stream);
}

extern "C" int fiber_intersect_nearest(const fiber_ray* rays, int64_t n_rays,
                                       const fiber_segments* segs, const fiber_pair* pairs,
                                       int64_t n_pairs, int max_depth, fiber_hit* hits,
                                       uint64_t* nearest, void* cuda_stream) {
  if (n_pairs > 0 && !nearest) return set_error(FIBER_EINVAL, "fiber_intersect_nearest: NULL nearest");
  return launch_intersect(rays, n_rays, segs, pairs, n_pairs, max_depth, hits, nearest, nullptr,
                          cuda_stream);
}

// For the library's own callers (grid.cu): mode bit 0 = closest, bit 1 = segment keys.
int launch_intersect_mode(const fiber_ray* rays, int64_t n_rays, const fiber_segments* segs,
                          const fiber_pair* pairs, int64_t n_pairs, int max_depth,
                          uint64_t* nearest, void* stream, int mode) {
  return launch_intersect(rays, n_rays, segs, pairs, n_pairs, max_depth, nullptr, nearest,
                          nullptr, stream, mode);
}

extern "C" int fiber_intersect_closest(const fiber_ray* rays, int64_t n_rays,
                                       const fiber_segments* segs, const fiber_pair* pairs,
                                       int64_t n_pairs, int max_depth, fiber_hit* hits,
                                       uint64_t* nearest, void* cuda_stream) {
  if (n_pairs > 0 && !nearest) return set_error(FIBER_EINVAL, "fiber_intersect_closest: NULL nearest");
  return launch_intersect(rays, n_rays, segs, pairs, n_pairs, max_depth, hits, nearest, nullptr,
                          cuda_stream, 1);
}

extern "C" int fiber_intersect_ex(const fiber_ray* rays, int64_t n_rays,
                                  const fiber_segments* segs, const fiber_pair* pairs,
                                  int64_t n_pairs, int max_depth, fiber_hit* hits,
                                  uint64_t* nearest, void* event_after_traverse,
                                  void* cuda_stream) {
  if (n_pairs > 0 && !hits && !nearest)
    return set_error(FIBER_EINVAL, "fiber_intersect_ex: NULL hits and nearest");
  return launch_intersect(rays, n_rays, segs, pairs, n_pairs, max_depth, hits, nearest,
                          event_after_traverse, cuda_stream);
}

extern "C" int fiber_nearest_init(uint64_t* nearest, int64_t n_rays, void* cuda_stream) {
  if (n_rays < 0 || (n_rays > 0 && !nearest))
    return set_error(FIBER_EINVAL, "fiber_nearest_init: bad arguments");
  int rc = check_device();
  if (rc != FIBER_OK) return rc;
  if (n_rays == 0) return FIBER_OK;
  int64_t blocks = (n_rays + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  fill_u64<<<(unsigned)blocks, 256, 0, (cudaStream_t)cuda_stream>>>(
      (unsigned long long*)nearest, n_rays, ~0ull);
  return check_launch("fiber_nearest_init");
}

// fiber_device.cuh -- device building blocks of the sm_100a ray/fiber path.
//
// Method: Binder & Keller, arXiv 1811.03374. Each function cites the passage it
// implements; DESIGN.md "Kernel" explains what differs from the paper's listings and why.
//
// Split of precision:
//   a2 setup      FP32 frame whose origin shift is formed in FP64 (intersect.cu).
//   a3-a6 loop    FP32: node test / descend / backtrack, the paper's hot loop (this file).
//   a7 finalise   FP64: re-solve of the accepted leaf (intersect.cu, kernel K3).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "fiber.h"

namespace fiberx {

// Bounds checks of the checking build (-DFIBER_CHECKS, `python -m paper_1811_03374_b200.build
// --variants` -> libfiber_checks.so): every index the kernels form is tested and a violation
// traps with its location.  compute-sanitizer is closed on this GPU pool, so the GPU suite is
// run against this build instead (scripts/run_checks.sh).  The product build compiles them out.
#ifdef FIBER_CHECKS
#define FIBER_CHECK(cond)                                                                  \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("FIBER_CHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__,    \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                                 \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define FIBER_CHECK(cond) \
  do {                    \
  } while (0)
#endif

// ------------------------------------------------------------------------------------
// small FP32 vector helpers (float4 = (x, y, z, w); w is the radius component)
// ------------------------------------------------------------------------------------
__device__ __forceinline__ float4 f4(float x, float y, float z, float w) {
  return make_float4(x, y, z, w);
}
// Packed FP32 (sm_100 FFMA2 / FADD2 / FMUL2): one issue slot for two lanes' worth of the
// float4 arithmetic of the descent; a scalar operand is broadcast by the instruction.
// -DFIBER_NO_PACKED builds the scalar form (a test build).
#ifndef FIBER_NO_PACKED
#define FIBER_PACKED 1
__device__ __forceinline__ float2 lo2(float4 a) { return make_float2(a.x, a.y); }
__device__ __forceinline__ float2 hi2(float4 a) { return make_float2(a.z, a.w); }
__device__ __forceinline__ float4 cat2(float2 a, float2 b) { return make_float4(a.x, a.y, b.x, b.y); }
__device__ __forceinline__ float2 s2(float s) { return make_float2(s, s); }
// a * b + c, a a scalar
__device__ __forceinline__ float4 fma4(float a, float4 b, float4 c) {
  return cat2(__ffma2_rn(s2(a), lo2(b), lo2(c)), __ffma2_rn(s2(a), hi2(b), hi2(c)));
}
__device__ __forceinline__ float4 mul4(float a, float4 b) {
  return cat2(__fmul2_rn(s2(a), lo2(b)), __fmul2_rn(s2(a), hi2(b)));
}
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return cat2(__fadd2_rn(lo2(a), lo2(b)), __fadd2_rn(hi2(a), hi2(b)));
}
__device__ __forceinline__ float4 sub4(float4 a, float4 b) {
  return cat2(__ffma2_rn(s2(-1.0f), lo2(b), lo2(a)), __ffma2_rn(s2(-1.0f), hi2(b), hi2(a)));
}
#endif

// float4 arithmetic: packed where available (fma(-1, b, a) rounds exactly as a - b)
__device__ __forceinline__ float4 operator+(float4 a, float4 b) {
#ifdef FIBER_PACKED
  return add4(a, b);
#else
  return f4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
#endif
}
__device__ __forceinline__ float4 operator-(float4 a, float4 b) {
#ifdef FIBER_PACKED
  return sub4(a, b);
#else
  return f4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w);
#endif
}
__device__ __forceinline__ float4 operator*(float s, float4 a) {
#ifdef FIBER_PACKED
  return mul4(s, a);
#else
  return f4(s * a.x, s * a.y, s * a.z, s * a.w);
#endif
}
__device__ __forceinline__ float dot3(float4 a, float4 b) {
  return fmaf(a.x, b.x, fmaf(a.y, b.y, a.z * b.z));
}
__device__ __forceinline__ float cross_norm2(float4 a, float4 b) {
  float cx = a.y * b.z - a.z * b.y;
  float cy = a.z * b.x - a.x * b.z;
  float cz = a.x * b.y - a.y * b.x;
  return fmaf(cx, cx, fmaf(cy, cy, cz * cz));
}

// Approximate MUFU intrinsics (<= 2 ulp); the parity tolerances absorb them.
// -DFIBER_IEEE_MATH builds the IEEE-rounded variant (a test build, never the product).
#ifdef FIBER_IEEE_MATH
__device__ __forceinline__ float fsqrt(float x) { return __fsqrt_rn(x); }
__device__ __forceinline__ float frcp(float x) { return __frcp_rn(x); }
__device__ __forceinline__ float fdiv(float a, float b) { return __fdiv_rn(a, b); }
#else
// .ftz: operands here are never subnormal (coordinates are normalised by the frame shift),
// and flushing drops the range fix-ups the non-ftz forms compile to.
__device__ __forceinline__ float fsqrt(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float frcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fdiv(float a, float b) { return a * frcp(b); }
#endif
// 1/sqrt(x) to ~1 ulp: the MUFU seed and one Newton step (unit ray directions, a2 setup)
__device__ __forceinline__ float frsqrt(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y * fmaf(-0.5f * x * y, y, 1.5f);
}

// ------------------------------------------------------------------------------------
// Curve in the (p, d, t0, t1) representation of 3.1, FP32.
// ------------------------------------------------------------------------------------
struct Delta {
  float4 p, d, t0, t1;
};

// The ray-frame curve kept for recomputation after backtracking, stored as the
// first point and the three hodograph differences D_k = P_{k+1} - P_k.
struct Hodo {
  float4 L0, D0, D1, D2;
};

// Blossom of the hodograph quadratic, H(a, b) = B(a, b, 1) - B(a, b, 0) = C'/3 blossomed:
// H(u, u) is the listing's eval_derivative.
__device__ __forceinline__ float4 hblossom(const Hodo& c, float a, float b) {
  float wa = (1.0f - a) * (1.0f - b), wb = fmaf(a, 1.0f - b, (1.0f - a) * b), wc = a * b;
  return f4(fmaf(wa, c.D0.x, fmaf(wb, c.D1.x, wc * c.D2.x)),
            fmaf(wa, c.D0.y, fmaf(wb, c.D1.y, wc * c.D2.y)),
            fmaf(wa, c.D0.z, fmaf(wb, c.D1.z, wc * c.D2.z)),
            fmaf(wa, c.D0.w, fmaf(wb, c.D1.w, wc * c.D2.w)));
}

// Re-calculation of the node curve on [u0, u1] after backtracking (lst:recalculation
// P:1371-1385).  The listing forms d = eval(u1) - eval(u0), which cancels catastrophically
// at depth (|d| ~ 2^-D); here every difference is a blossom of the hodograph times
// h = u1 - u0 (exact), so d, t0, t1 keep full relative precision:
//   p = C(u0) = L0 + u0 (H(0,0) + H(0,u0) + H(u0,u0)),  t0 = h H(u0,u0),  t1 = h H(u1,u1),
//   d = h (H(u0,u0) + H(u0,u1) + H(u1,u1)).
__device__ __forceinline__ void recompute(const Hodo& c, float u0, float u1, Delta& cur) {
  float h = u1 - u0;
  float4 H00 = hblossom(c, u0, u0), H01 = hblossom(c, u0, u1), H11 = hblossom(c, u1, u1);
  float4 H0u = hblossom(c, 0.0f, u0);
  float4 s = c.D0 + H0u + H00;
  cur.p = f4(fmaf(u0, s.x, c.L0.x), fmaf(u0, s.y, c.L0.y), fmaf(u0, s.z, c.L0.z),
             fmaf(u0, s.w, c.L0.w));
  cur.t0 = h * H00;
  cur.t1 = h * H11;
  cur.d = h * (H00 + H01 + H11);
}

// Interval (start, size) in 2^-23 units -> [u0, u1] (lst:calculate_interval P:1331-1345).
__device__ __forceinline__ void get_interval(uint32_t start, uint32_t size, float& u0, float& u1) {
  uint32_t ui0 = 0x3f800000u | start;
  u0 = __uint_as_float(ui0) - 1.0f;
  uint32_t ui1 = min(ui0 + size, 0x40000000u);
  u1 = __uint_as_float(ui1) - 1.0f;
}

// Which constraint bounds t_min (F6, R7).  Every cropping plane -- the slab
// planes of lst:calc_t_interval and the partition planes of P:1441-1442 -- is the normal
// plane of the curve at a dyadic parameter u (through C(u), normal parallel to C'(u)), so
// the tag is that u in 2^-23 units (0 = the start cap, 2^23 = the end cap); TAG_ORIGIN
// marks the ray origin bound t >= 0.  K3 re-solves crop-plane entries in FP64 from it.
constexpr uint32_t TAG_ORIGIN = 0xffffffffu;

// The node's own slab: [lo0, hi0] cut by the start plane (through p, normal t0, keeps
// <x - p, t0> >= 0) and the end plane (through p + d, normal t1, keeps <x - p - d, t1> <= 0)
// -- lst:calc_t_interval P:1459-1477 with F3 (a plane parallel to the ray keeps all or
// nothing) and F7 (t_max passed explicitly).  tag: what bounds t_min.  `widen` moves the
// two planes outward by a bound on their FP32 rounding error: used after a node was
// RE-COMPUTED (lst:recalculation), whose planes can sit a few ulps off the ones the
// sibling's interval was cut with; without it a hit on the shared plane could fall into
// the gap between the two intervals.
__device__ __forceinline__ void slab(const Delta& c, float lo0, float hi0, uint32_t u0tag,
                                     uint32_t u1tag, float& tmin, float& tmax, uint32_t& tag,
                                     bool widen = false, float* kappa = nullptr) {
  tmin = lo0;
  tmax = hi0;
  tag = TAG_ORIGIN;
  float n0 = dot3(c.t0, c.p), z0 = c.t0.z;
  float4 e = c.p + c.d;
  float n1 = dot3(c.t1, e), z1 = c.t1.z;
  if (widen) {
    // |error of <t, x>| <~ 2^-20 (|t| . |x|) covers the dot product and the recomputed x
    const float k = 9.5367431640625e-07f;  // 2^-20
    float a0 = fmaf(fabsf(c.t0.x), fabsf(c.p.x), fmaf(fabsf(c.t0.y), fabsf(c.p.y), fabsf(c.t0.z) * fabsf(c.p.z)));
    float a1 = fmaf(fabsf(c.t1.x), fabsf(e.x), fmaf(fabsf(c.t1.y), fabsf(e.y), fabsf(c.t1.z) * fabsf(e.z)));
    n0 -= k * a0;  // start plane moved against t0 (outward)
    n1 += k * a1;  // end plane moved along t1 (outward)
  }
  if (z0 > 0.0f) {
    float x = fdiv(n0, z0);
    if (x > tmin) tmin = x, tag = u0tag;
  } else if (z0 < 0.0f) {
    tmax = fminf(tmax, fdiv(n0, z0));
  } else if (n0 > 0.0f) {
    tmin = INFINITY;  // parallel and on the invalid side: empty
  }
  if (z1 < 0.0f) {
    float x = fdiv(n1, z1);
    if (x > tmin) tmin = x, tag = u1tag;
  } else if (z1 > 0.0f) {
    tmax = fminf(tmax, fdiv(n1, z1));
  } else if (n1 < 0.0f) {
    tmin = INFINITY;
  }
  if (kappa) {  // conditioning of the two crossings: |t|_1 / |t_z| (>= 1 / cos)
    float k0 = (fabsf(c.t0.x) + fabsf(c.t0.y) + fabsf(z0)) * frcp(fabsf(z0));
    float k1 = (fabsf(c.t1.x) + fabsf(c.t1.y) + fabsf(z1)) * frcp(fabsf(z1));
    *kappa = fminf(fmaxf(k0, k1), 1e30f);
  }
}

// Descent-time crop limit: partition planes crop the ray interval
// only down to level kCropLevel.  Below it a level's slab along the ray (~2^-l of the
// segment) falls under FP32 resolution of the plane crossings, so its bounds would invert
// by rounding; deeper nodes inherit the level-kCropLevel interval, and the planes still
// order the children.  The FP64 finalisation then re-solves the exact leaf.
#ifndef FIBER_CROP_LEVEL
#define FIBER_CROP_LEVEL 12
#endif
constexpr int kCropLevel = FIBER_CROP_LEVEL;
constexpr uint32_t kCropMinSize = 1u << (FIBER_MAX_DEPTH - kCropLevel);

// Node test (a3): conservative radius (lst:calc_radius P:1415-1425 with the point-line
// distance of lst:distance-point-line P:1308-1328, here |t x d|^2 / |d|^2) and the unit ray
// x infinite cylinder of App. A (lst:ray-cylinder P:1279-1303, eq. P:814, t_cpa P:825-833,
// s P:862-866).  F4: an axis parallel to the ray gives the whole line if inside.  F5: a
// miss is reported as `false`, never as a sentinel interval.
__device__ __forceinline__ bool cylinder(const Delta& c, float& c0, float& c1, float* tie_e = nullptr,
                                         float* inv_sin = nullptr, float delta = 0.0f) {
  float dd = dot3(c.d, c.d);
  float m2 = fmaxf(cross_norm2(c.t0, c.d), cross_norm2(c.t1, c.d));
  float dist = fsqrt(m2 * frcp(dd));
  float maxr = c.p.w + fmaxf(fmaxf(0.0f, c.t0.w), fmaxf(c.d.w, c.d.w - c.t1.w));
  float R = dist + maxr;
  float g = fmaf(c.d.x, c.d.x, c.d.y * c.d.y);
  float h = frcp(g);
  float dxy = fmaf(c.d.x, c.p.y, -c.d.y * c.p.x);
  float e = fmaf(R, R, -dxy * dxy * h);
  float tc = fmaf(-c.d.z * h, fmaf(c.d.x, c.p.x, c.d.y * c.p.y), c.p.z);
  float s = fsqrt(e * fmaf(c.d.z, c.d.z, g) * h);
  // F4 (selects, no branch): axis parallel to the ray -> whole line if inside, else empty
  bool par = g <= 1e-12f * dd;
  bool in = fmaf(c.p.x, c.p.x, c.p.y * c.p.y) <= R * R;
  c0 = par ? -INFINITY : tc - s;
  c1 = par ? INFINITY : tc + s;
  if (tie_e) {
    // near-tie of the distance test |R - dist| against the error of FP32 coordinates
    // (delta) and a relative 2^-16 (R5): flags the pair for the FP64 re-run
    float ee = par ? fmaf(R, R, -fmaf(c.p.x, c.p.x, c.p.y * c.p.y)) : e;
    *tie_e = fabsf(ee) - R * fmaf(1.52587890625e-05f, R, 2.0f * delta);  // < 0: tie
    *inv_sin = fsqrt(dd * h);                                        // 1 / sin(ray, axis)
  }
  return par ? in : (e >= 0.0f);
}

// Descend (a4): split point and tangent of 3.1, partition plane through
// p + delta_p with normal t_c (lst:ray-plane P:1246-1251), near child first
// (P:1444 as XOR, F9), both-hit on the uncropped cylinder interval,
// one-bound update while `crop`.  F3: a partition plane parallel to the
// ray: near child = the side of the ray, no both, no update.  The children follow the
// delta rules of lst:subdivide P:1391-1412:
//   left = (p, dp, t0/2, t_c),   right = (p + dp, d - dp, t_c, t1/2).
struct Split {
  float4 dp, tcn, S;
};

// Split point and tangent of node c (3.1): delta_p, t_c and S = p + delta_p.
__device__ __forceinline__ void split_geometry(const Delta& c, Split& sp) {
#ifdef FIBER_PACKED
  sp.dp = fma4(0.375f, sub4(c.t0, c.t1), mul4(0.5f, c.d));
  sp.tcn = fma4(-0.125f, add4(c.t0, c.t1), mul4(0.25f, c.d));
  sp.S = add4(c.p, sp.dp);
#else
  sp.dp = 0.375f * (c.t0 - c.t1) + 0.5f * c.d;
  sp.tcn = 0.25f * c.d - 0.125f * (c.t0 + c.t1);
  sp.S = c.p + sp.dp;
#endif
}

// The child on side `right` of the split.  Packed form: blends with r = 0 / 1 that are
// exact for finite operands (x + 0 y = x, 0 x + y = y, 1 x + y = fl(x + y)), so the child
// equals the selected one up to the sign of a zero:
//   p'  = p + r dp,   d' = (1 - 2r) dp + r d,
//   t0' = (1-r)/2 t0 + r t_c,   t1' = r/2 t1 + (1 - r) t_c.
__device__ __forceinline__ void child(const Delta& c, const Split& sp, bool right, Delta& out) {
#ifdef FIBER_PACKED
  const float r = right ? 1.0f : 0.0f, nr = 1.0f - r;
  out.p = fma4(r, sp.dp, c.p);
  out.d = fma4(fmaf(-2.0f, r, 1.0f), sp.dp, mul4(r, c.d));
  out.t0 = fma4(0.5f * nr, c.t0, mul4(r, sp.tcn));
  out.t1 = fma4(0.5f * r, c.t1, mul4(nr, sp.tcn));
#else
#define FX_SEL4(dst, a, b)                                                             \
  dst = make_float4(right ? (a).x : (b).x, right ? (a).y : (b).y, right ? (a).z : (b).z, \
                    right ? (a).w : (b).w)
  float4 rd = c.d - sp.dp, h0 = 0.5f * c.t0, h1 = 0.5f * c.t1;
  FX_SEL4(out.p, sp.S, c.p);
  FX_SEL4(out.d, rd, sp.dp);
  FX_SEL4(out.t0, sp.tcn, h0);
  FX_SEL4(out.t1, h1, sp.tcn);
#undef FX_SEL4
#endif
}

}  // namespace fiberx

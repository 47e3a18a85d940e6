// fiber_device.cuh -- device building blocks of the sm_100a ray/fiber path.
//
// Method: Binder & Keller, arXiv 1811.03374. Each function cites the passage it
// implements; DESIGN.md "Kernel" explains what differs from the paper's listings and why.
//
// Split of precision:
//   a2 setup      FP64: origin shifted onto the ray next to the segment, ONB, transform to
//                 the unit-ray frame, rounded once to FP32.
//   a3-a6 loop    FP32: node test / descend / backtrack, the paper's hot loop.
//   a7 finalise   FP64: re-solve of the accepted leaf (walking to the neighbour leaf the
//                 ray really enters when FP32 picked a neighbour at D >= 18).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "fiber.h"

namespace fiberx {

// ------------------------------------------------------------------------------------
// small FP32 vector helpers (float4 = (x, y, z, w); w is the radius component)
// ------------------------------------------------------------------------------------
__device__ __forceinline__ float4 f4(float x, float y, float z, float w) {
  return make_float4(x, y, z, w);
}
__device__ __forceinline__ float4 operator+(float4 a, float4 b) {
  return f4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float4 operator-(float4 a, float4 b) {
  return f4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w);
}
__device__ __forceinline__ float4 operator*(float s, float4 a) {
  return f4(s * a.x, s * a.y, s * a.z, s * a.w);
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

// ------------------------------------------------------------------------------------
// FP64 helpers
// ------------------------------------------------------------------------------------
struct d3 {
  double x, y, z;
};
struct d4 {
  double x, y, z, w;
};
__device__ __forceinline__ d3 mk3(double x, double y, double z) { return d3{x, y, z}; }
__device__ __forceinline__ d3 sub(d3 a, d3 b) { return d3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ double dot(d3 a, d3 b) {
  return fma(a.x, b.x, fma(a.y, b.y, a.z * b.z));
}
__device__ __forceinline__ d4 add4(d4 a, d4 b) { return d4{a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w}; }
__device__ __forceinline__ d4 sub4(d4 a, d4 b) { return d4{a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w}; }
__device__ __forceinline__ d4 mul4(double s, d4 a) { return d4{s * a.x, s * a.y, s * a.z, s * a.w}; }
__device__ __forceinline__ d4 fma4(double s, d4 a, d4 b) {
  return d4{fma(s, a.x, b.x), fma(s, a.y, b.y), fma(s, a.z, b.z), fma(s, a.w, b.w)};
}
__device__ __forceinline__ float4 to_f4(d4 a) {
  return make_float4((float)a.x, (float)a.y, (float)a.z, (float)a.w);
}

// Orthonormal basis around a unit vector w: Duff et al. 2017's revision of Frisvad's
// construction, named by the paper at P:476-477 (the listing calls make_ONB).
__device__ __forceinline__ void make_onb(d3 w, d3& b1, d3& b2) {
  double sign = copysign(1.0, w.z);
  double a = -1.0 / (sign + w.z);
  double b = w.x * w.y * a;
  b1 = mk3(1.0 + sign * w.x * w.x * a, sign * b, -sign * w.x);
  b2 = mk3(b, sign + w.y * w.y * a, -w.y);
}

// ------------------------------------------------------------------------------------
// Per-pair frame (a2).  World point X maps to local (<X-o', b1>, <X-o', b2>, <X-o', w^>)
// with o' = o + ts w^ on the ray next to the segment (ts = <c - o, w^>, c = (P0 + P3)/2):
// the ray becomes the unit ray (0,0,0) + s (0,0,1) of P:475-481, and local coordinates are
// small, so their FP32 rounding is relative to the segment size, not to |o - P|.
// ------------------------------------------------------------------------------------
struct Frame {
  d3 o;        // o' (world)
  d3 b1, b2, w;  // orthonormal frame, w = d / |d|
  double ts;   // o' = o + ts * w (distance units)
  double lw;   // |d|: t = s / |d|
};

// Returns false for a degenerate ray (non-finite values, zero direction, tmax <= 0).
__device__ __forceinline__ bool make_frame(const float4 ray0, const float4 ray1, const float4 P0,
                                           const float4 P3, Frame& F) {
  d3 o = mk3(ray0.x, ray0.y, ray0.z);
  d3 d = mk3(ray1.x, ray1.y, ray1.z);
  double lw = sqrt(dot(d, d));
  bool ok = isfinite(ray0.x) && isfinite(ray0.y) && isfinite(ray0.z) && isfinite(ray1.x) &&
            isfinite(ray1.y) && isfinite(ray1.z) && !(ray0.w <= 0.0f) && !isnan(ray0.w) &&
            lw > 0.0;
  if (!ok) lw = 1.0, d = mk3(0, 0, 1);
  double il = 1.0 / lw;
  F.w = mk3(d.x * il, d.y * il, d.z * il);
  F.lw = lw;
  make_onb(F.w, F.b1, F.b2);
  d3 c = mk3(0.5 * ((double)P0.x + (double)P3.x), 0.5 * ((double)P0.y + (double)P3.y),
             0.5 * ((double)P0.z + (double)P3.z));
  F.ts = dot(sub(c, o), F.w);
  F.o = mk3(fma(F.ts, F.w.x, o.x), fma(F.ts, F.w.y, o.y), fma(F.ts, F.w.z, o.z));
  return ok;
}

__device__ __forceinline__ d4 to_local(const Frame& F, float4 P) {
  d3 q = sub(mk3(P.x, P.y, P.z), F.o);
  return d4{dot(q, F.b1), dot(q, F.b2), dot(q, F.w), (double)P.w};
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

// Bound tags (which constraint set t_min), F6.
enum : uint32_t { TAG_ORIGIN = 0, TAG_START = 1, TAG_END = 2, TAG_INTERNAL = 3 };

// The node's own slab: [lo0, hi0] cut by the start plane (through p, normal t0, keeps
// <x - p, t0> >= 0) and the end plane (through p + d, normal t1, keeps <x - p - d, t1> <= 0)
// -- lst:calc_t_interval P:1459-1477 with F3 (a plane parallel to the ray keeps all or
// nothing) and F7 (t_max passed explicitly).  tag: what bounds t_min.
__device__ __forceinline__ void slab(const Delta& c, float lo0, float hi0, bool u0_is_0,
                                     bool u1_is_1, float& tmin, float& tmax, uint32_t& tag) {
  tmin = lo0;
  tmax = hi0;
  tag = TAG_ORIGIN;
  float n0 = dot3(c.t0, c.p), z0 = c.t0.z;
  float4 e = c.p + c.d;
  float n1 = dot3(c.t1, e), z1 = c.t1.z;
  if (z0 > 0.0f) {
    float x = n0 / z0;
    if (x > tmin) tmin = x, tag = u0_is_0 ? TAG_START : TAG_INTERNAL;
  } else if (z0 < 0.0f) {
    tmax = fminf(tmax, n0 / z0);
  } else if (n0 > 0.0f) {
    tmin = INFINITY;  // parallel and on the invalid side: empty
  }
  if (z1 < 0.0f) {
    float x = n1 / z1;
    if (x > tmin) tmin = x, tag = u1_is_1 ? TAG_END : TAG_INTERNAL;
  } else if (z1 > 0.0f) {
    tmax = fminf(tmax, n1 / z1);
  } else if (n1 < 0.0f) {
    tmin = INFINITY;
  }
}

// Node test (a3): conservative radius (lst:calc_radius P:1415-1425 with the point-line
// distance of lst:distance-point-line P:1308-1328, here |t x d|^2 / |d|^2) and the unit ray
// x infinite cylinder of App. A (lst:ray-cylinder P:1279-1303, eq. P:814, t_cpa P:825-833,
// s P:862-866).  F4: an axis parallel to the ray gives the whole line if inside.  F5: a
// miss is reported as `false`, never as a sentinel interval.
__device__ __forceinline__ bool cylinder(const Delta& c, float& c0, float& c1) {
  float dd = dot3(c.d, c.d);
  float m2 = fmaxf(cross_norm2(c.t0, c.d), cross_norm2(c.t1, c.d));
  float dist = sqrtf(m2 / dd);
  float maxr = c.p.w + fmaxf(fmaxf(0.0f, c.t0.w), fmaxf(c.d.w, c.d.w - c.t1.w));
  float R = dist + maxr;
  float g = fmaf(c.d.x, c.d.x, c.d.y * c.d.y);
  if (g <= 1e-12f * dd) {
    c0 = -INFINITY;
    c1 = INFINITY;
    return fmaf(c.p.x, c.p.x, c.p.y * c.p.y) <= R * R;
  }
  float h = 1.0f / g;
  float dxy = c.d.x * c.p.y - c.d.y * c.p.x;
  float e = fmaf(R, R, -dxy * dxy * h);
  float tc = c.p.z - c.d.z * fmaf(c.d.x, c.p.x, c.d.y * c.p.y) * h;
  float s = sqrtf(e * fmaf(c.d.z, c.d.z, g) * h);
  c0 = tc - s;
  c1 = tc + s;
  return e >= 0.0f;
}

// Descend (a4): split point and tangent of 3.1, partition plane through
// p + delta_p with normal t_c (lst:ray-plane P:1246-1251), near child first
// (P:1444 as XOR, F9), both-hit on the uncropped cylinder interval,
// one-bound update, child by the delta rules (lst:subdivide P:1391-1412).
// F3: a partition plane parallel to the ray: near child = the side of the ray, no both,
// no update.
__device__ __forceinline__ void descend(Delta& c, float c0, float c1, float& tmin, float& tmax,
                                        uint32_t& tag, bool& right, bool& both) {
  float4 dp = 0.375f * (c.t0 - c.t1) + 0.5f * c.d;
  float4 tcn = 0.25f * c.d - 0.125f * (c.t0 + c.t1);
  float4 S = c.p + dp;
  float num = dot3(tcn, S), nz = tcn.z;
  if (nz != 0.0f) {
    float tP = num / nz;
    right = (tP > c0) != (nz > 0.0f);
    both = (c0 < tP) && (tP < c1);
    if (tP > c0) {
      tmax = fminf(tmax, tP);
    } else if (tP > tmin) {
      tmin = tP;
      tag = TAG_INTERNAL;
    }
  } else {
    right = num < 0.0f;
    both = false;
  }
  if (right) {
    c.p = S;
    c.d = c.d - dp;
    c.t0 = tcn;
    c.t1 = 0.5f * c.t1;
  } else {
    c.d = dp;
    c.t0 = 0.5f * c.t0;
    c.t1 = tcn;
  }
}

// ------------------------------------------------------------------------------------
// Octahedral normal encoding, 2 x snorm16 (decode error < 6e-5 rad).
// ------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t encode_oct(double nx, double ny, double nz) {
  double l1 = fabs(nx) + fabs(ny) + fabs(nz);
  if (!(l1 > 0.0)) return 0u;
  double x = nx / l1, y = ny / l1;
  if (nz < 0.0) {
    double ox = (1.0 - fabs(y)) * copysign(1.0, x);
    double oy = (1.0 - fabs(x)) * copysign(1.0, y);
    x = ox;
    y = oy;
  }
  int ix = __double2int_rn(fmin(1.0, fmax(-1.0, x)) * 32767.0);
  int iy = __double2int_rn(fmin(1.0, fmax(-1.0, y)) * 32767.0);
  return ((uint32_t)ix & 0xffffu) | (((uint32_t)iy & 0xffffu) << 16);
}

}  // namespace fiberx

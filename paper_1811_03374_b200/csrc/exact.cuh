// exact.cuh -- the traversal in FP64 (run by kernel K3), for the pairs the FP32 traversal (K2)
// flagged as decided by a near-tie (R5).
//
// The same algorithm as K2 (lst:algorithm P:1591-1651 with F1-F9), written in double: the
// unit-ray frame of P:475-483 built in FP64 (Duff et al.'s ONB) with its origin
// on the ray next to the segment, the App. A cylinder, partition planes cropping at every
// level, and re-calculation (lst:recalculation P:1371-1385) after every backtrack.  Its
// decisions then agree with the FP64 definition except within ~1e-15 of a tie, so hit
// flags are exact outside the north star's 1e-6 r band.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "fiber.h"

namespace fiberx {
namespace exact {

// Double-precision reciprocal, division and square root from the MUFU seeds
// (rcp/rsqrt.approx.f64) refined by Newton steps: ~1 ulp, and a short dependency chain
// instead of the IEEE division/sqrt sequences (a re-run is one lane's latency-bound chain).
// rcp64 takes two steps.
__device__ __forceinline__ double rcp64(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r);
  return fma(r, fma(-x, r, 1.0), r);
}
// The seeds are good to 2^-20 (measured on B200: scripts/micro/seed.cu).  One Newton step
// gives ~1e-12; the residual correction that ends div64 and sqrt64 squares that error, so
// both need only one step before it.
__device__ __forceinline__ double div64(double a, double b) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  r = fma(r, fma(-b, r, 1.0), r);
  const double q = a * r;
  return fma(r, fma(-b, q, a), q);  // one residual correction
}
__device__ __forceinline__ double sqrt64(double x) {
  if (!(x > 0.0)) return x == 0.0 ? 0.0 : sqrt(x);
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-0.5 * x * y, y, 1.5);
  const double s = x * y;
  return fma(0.5 * y, fma(-s, s, x), s);
}

struct V4 {
  double x, y, z, w;
};
__device__ __forceinline__ V4 v4(double x, double y, double z, double w) { return V4{x, y, z, w}; }
__device__ __forceinline__ V4 add(V4 a, V4 b) { return v4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
__device__ __forceinline__ V4 sub(V4 a, V4 b) { return v4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w); }
__device__ __forceinline__ V4 scl(double s, V4 a) { return v4(s * a.x, s * a.y, s * a.z, s * a.w); }
__device__ __forceinline__ double dot3(V4 a, V4 b) { return fma(a.x, b.x, fma(a.y, b.y, a.z * b.z)); }
__device__ __forceinline__ double crossn2(V4 a, V4 b) {
  double cx = fma(a.y, b.z, -a.z * b.y), cy = fma(a.z, b.x, -a.x * b.z), cz = fma(a.x, b.y, -a.y * b.x);
  return fma(cx, cx, fma(cy, cy, cz * cz));
}

struct Curve {
  V4 p, d, t0, t1;  // (p, d, t0, t1) of 3.1
};
struct Hodo64 {
  V4 L0, D0, D1, D2;
};

__device__ __forceinline__ V4 hb(const Hodo64& c, double a, double b) {
  double wa = (1.0 - a) * (1.0 - b), wb = a * (1.0 - b) + (1.0 - a) * b, wc = a * b;
  return v4(fma(wa, c.D0.x, fma(wb, c.D1.x, wc * c.D2.x)), fma(wa, c.D0.y, fma(wb, c.D1.y, wc * c.D2.y)),
            fma(wa, c.D0.z, fma(wb, c.D1.z, wc * c.D2.z)), fma(wa, c.D0.w, fma(wb, c.D1.w, wc * c.D2.w)));
}

// node curve on [u0, u1] from the hodograph blossoms (lst:recalculation)
__device__ __forceinline__ Curve node(const Hodo64& c, double u0, double u1) {
  double h = u1 - u0;
  V4 H00 = hb(c, u0, u0), H01 = hb(c, u0, u1), H11 = hb(c, u1, u1), H0u = hb(c, 0.0, u0);
  V4 s = add(add(c.D0, H0u), H00);
  Curve q;
  q.p = v4(fma(u0, s.x, c.L0.x), fma(u0, s.y, c.L0.y), fma(u0, s.z, c.L0.z), fma(u0, s.w, c.L0.w));
  q.t0 = scl(h, H00);
  q.t1 = scl(h, H11);
  q.d = scl(h, add(add(H00, H01), H11));
  return q;
}

constexpr uint32_t kOrigin = 0xffffffffu;

// own slab, lst:calc_t_interval with F3/F7; tags are the planes' u (see fiber_device.cuh)
__device__ __forceinline__ void slab(const Curve& c, double lo0, double hi0, uint32_t u0tag,
                                     uint32_t u1tag, double& tmin, double& tmax, uint32_t& tag) {
  tmin = lo0;
  tmax = hi0;
  tag = kOrigin;
  double n0 = dot3(c.t0, c.p), z0 = c.t0.z;
  V4 e = add(c.p, c.d);
  double n1 = dot3(c.t1, e), z1 = c.t1.z;
  if (z0 > 0.0) {
    double x = div64(n0, z0);
    if (x > tmin) tmin = x, tag = u0tag;
  } else if (z0 < 0.0) {
    tmax = fmin(tmax, div64(n0, z0));
  } else if (n0 > 0.0) {
    tmin = INFINITY;
  }
  if (z1 < 0.0) {
    double x = div64(n1, z1);
    if (x > tmin) tmin = x, tag = u1tag;
  } else if (z1 > 0.0) {
    tmax = fmin(tmax, div64(n1, z1));
  } else if (n1 < 0.0) {
    tmin = INFINITY;
  }
}

// unit ray x conservative cylinder (App. A), F4 for an axis parallel to the ray
__device__ __forceinline__ bool cylinder(const Curve& c, double& c0, double& c1) {
  double g = fma(c.d.x, c.d.x, c.d.y * c.d.y);
  double dd = fma(c.d.z, c.d.z, g);
  double m2 = fmax(crossn2(c.t0, c.d), crossn2(c.t1, c.d));
  double R = sqrt64(m2 * rcp64(dd)) + c.p.w + fmax(fmax(0.0, c.t0.w), fmax(c.d.w, c.d.w - c.t1.w));
  if (g == 0.0) {
    c0 = -INFINITY;
    c1 = INFINITY;
    return fma(c.p.x, c.p.x, c.p.y * c.p.y) <= R * R;
  }
  const double ig = rcp64(g);
  double dxy = fma(c.d.x, c.p.y, -c.d.y * c.p.x);
  double e = fma(-dxy * dxy, ig, R * R);
  if (!(e >= 0.0)) return false;
  double tc = fma(-c.d.z * ig, fma(c.d.x, c.p.x, c.d.y * c.p.y), c.p.z);
  double s = sqrt64(e * dd * ig);
  c0 = tc - s;
  c1 = tc + s;
  return true;
}

struct Result {
  bool hit;
  uint32_t start, size, kind, inside, tag, tests, backtracks;
  double z;  // z* in the FP64 frame (not used by K3)
};

// The whole traversal of one pair in FP64.
__device__ __forceinline__ Result traverse(const float4 ray0, const float4 ray1, const float4 P0,
                                        const float4 P1, const float4 P2, const float4 P3,
                                        bool quad, int depth, uint32_t start0 = 0u,
                                        uint32_t size0 = 1u << FIBER_MAX_DEPTH,
                                        uint32_t bits0 = 0u) {
  Result res{false, 0, 0, 0, 0, kOrigin, 0, 0, 0.0};
  // frame: o' = o + ts w^ next to the segment, ONB (Duff et al.)
  double wx = ray1.x, wy = ray1.y, wz = ray1.z;
  const double lw = sqrt64(wx * wx + wy * wy + wz * wz);
  const double ilw = rcp64(lw);
  wx *= ilw;
  wy *= ilw;
  wz *= ilw;
  const double sign = copysign(1.0, wz);
  const double a = -rcp64(sign + wz), b = wx * wy * a;
  const V4 b1 = v4(1.0 + sign * wx * wx * a, sign * b, -sign * wx, 0.0);
  const V4 b2 = v4(b, sign + wy * wy * a, -wy, 0.0);
  const V4 W = v4(wx, wy, wz, 0.0);
  const V4 o = v4(ray0.x, ray0.y, ray0.z, 0.0);
  const V4 cm = v4(0.5 * ((double)P0.x + (double)P3.x), 0.5 * ((double)P0.y + (double)P3.y),
                   0.5 * ((double)P0.z + (double)P3.z), 0.0);
  const double ts = dot3(sub(cm, o), W);
  const V4 op = v4(fma(ts, wx, o.x), fma(ts, wy, o.y), fma(ts, wz, o.z), 0.0);
  auto loc = [&](float4 P) {
    V4 q = sub(v4(P.x, P.y, P.z, 0.0), op);
    return v4(dot3(q, b1), dot3(q, b2), dot3(q, W), (double)P.w);
  };
  const V4 L0 = loc(P0), L1 = loc(P1), L2 = loc(P2), L3 = loc(P3);
  // a quadratic (q0, q1, q2) = (P0, P1, P3) is degree-elevated exactly (fiber.h)
  const Hodo64 hc = quad ? Hodo64{L0, scl(2.0 / 3.0, sub(L1, L0)), scl(1.0 / 3.0, sub(L3, L0)),
                                  scl(2.0 / 3.0, sub(L3, L1))}
                         : Hodo64{L0, sub(L1, L0), sub(L2, L1), sub(L3, L2)};
  // ray interval [0, tmax) in local distance units
  const double lo0 = -ts, hi0 = (double)ray0.w * lw - ts;
  // resume at node (start0, size0) with the pending levels bits0 (the root by default): the
  // node's curve re-calculated and its interval from its own end planes, as after a
  // backtrack -- the carried interval of a descent equals it in exact
  // arithmetic
  const double inv23 = 1.0 / (double)(1u << FIBER_MAX_DEPTH);
  Curve cur = size0 == (1u << FIBER_MAX_DEPTH)
                  ? Curve{L0, sub(L3, L0), hc.D0, hc.D2}
                  : node(hc, (double)start0 * inv23, (double)(start0 + size0) * inv23);
  double tmin, tmax;
  uint32_t tag;
  slab(cur, lo0, hi0, start0, start0 + size0, tmin, tmax, tag);
  const uint32_t min_size = 1u << (FIBER_MAX_DEPTH - depth);
  uint32_t bits = bits0, size = size0, start = start0, tests = 0, bt = 0;
  while (true) {
    ++tests;
    double c0, c1;
    bool pass = cylinder(cur, c0, c1);
    pass = pass && c1 >= tmin && c0 <= tmax && tmin <= tmax;  // P:1618 + F1, F5
    if (pass) {
      if (size <= min_size) {  // leaf, F2
        res.z = fmax(c0, tmin);
        res.hit = res.z < hi0;
        res.kind = FIBER_KIND_LATERAL;
        if (!(c0 >= tmin)) {
          if (tag == kOrigin) res.inside = 1, res.kind = FIBER_KIND_WEDGE;
          else if (tag == 0u && start == 0u) res.kind = FIBER_KIND_CAP0;
          else if (tag == (1u << FIBER_MAX_DEPTH) && start + size == (1u << FIBER_MAX_DEPTH))
            res.kind = FIBER_KIND_CAP1;
          else res.kind = FIBER_KIND_WEDGE;
        }
        break;
      }
      // partition: split point, plane, near child, both, one-bound update
      V4 dp = add(scl(0.375, sub(cur.t0, cur.t1)), scl(0.5, cur.d));
      V4 tcn = sub(scl(0.25, cur.d), scl(0.125, add(cur.t0, cur.t1)));
      V4 S = add(cur.p, dp);
      double num = dot3(tcn, S), nz = tcn.z;
      bool right, both;
      if (nz != 0.0) {
        double tP = div64(num, nz);
        right = (tP > c0) != (nz > 0.0);
        both = (c0 < tP) && (tP < c1);
        if (tP > c0) tmax = fmin(tmax, tP);
        else if (tP > tmin) tmin = tP, tag = start + (size >> 1);
      } else {
        right = num < 0.0;
        both = false;
      }
      // the child as an exact blend with r = 0 / 1 (as K2's child(); no divergent copies of
      // the loop-carried curve): p' = p + r dp, d' = (1 - 2r) dp + r d,
      // t0' = (1-r)/2 t0 + r t_c, t1' = r/2 t1 + (1-r) t_c
      {
        const double r = right ? 1.0 : 0.0, nr = 1.0 - r, s = 1.0 - 2.0 * r;
        const double h0 = 0.5 * nr, h1 = 0.5 * r;
        auto blend = [](double a, V4 x, V4 y) {  // a x + y
          return v4(fma(a, x.x, y.x), fma(a, x.y, y.y), fma(a, x.z, y.z), fma(a, x.w, y.w));
        };
        const V4 d = cur.d;
        cur.p = blend(r, dp, cur.p);
        cur.d = blend(s, dp, scl(r, d));
        cur.t0 = blend(h0, cur.t0, scl(r, tcn));
        cur.t1 = blend(h1, cur.t1, scl(nr, tcn));
      }
      size >>= 1;
      if (both) bits |= size;
      if (right) start |= size;
    } else {
      if (bits == 0u) break;
      ++bt;
      size = bits & (0u - bits);  // jump_up
      start ^= size;
      bits ^= size;
      start &= ~(size - 1u);
      cur = node(hc, (double)start * inv23, (double)(start + size) * inv23);
      slab(cur, lo0, hi0, start, start + size, tmin, tmax, tag);
    }
  }
  res.start = start;
  res.size = size;
  res.tag = tag;
  res.tests = tests;
  res.backtracks = bt;
  return res;
}

}  // namespace exact
}  // namespace fiberx

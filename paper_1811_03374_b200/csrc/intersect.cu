// intersect.cu -- K2: the ray/fiber pair intersector for sm_100a, plus its C ABI.
//
// One thread per ray-segment pair, the stackless traversal of
// lst:algorithm with the readings F1-F9 of DESIGN.md.
// DESIGN.md "Kernel" describes the launch shape and precision split.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "fiber.h"
#include "fiber_device.cuh"
#include "fiber_internal.h"

namespace fiberx {

// ------------------------------------------------------------------------------------
// FP64 leaf geometry for finalisation (a7)
// ------------------------------------------------------------------------------------
struct LeafD {
  d4 p, d, t0, t1;
};

__device__ __forceinline__ d4 hblossom_d(const d4 D[3], double a, double b) {
  double wa = (1.0 - a) * (1.0 - b), wb = a * (1.0 - b) + (1.0 - a) * b, wc = a * b;
  return d4{wa * D[0].x + wb * D[1].x + wc * D[2].x, wa * D[0].y + wb * D[1].y + wc * D[2].y,
            wa * D[0].z + wb * D[1].z + wc * D[2].z, wa * D[0].w + wb * D[1].w + wc * D[2].w};
}

// Sub-curve on [u0, u1] of the local FP64 curve, in the (p, d, t0, t1) form (3.1).
__device__ __forceinline__ LeafD leaf_d(const d4 L[4], double u0, double u1) {
  d4 D[3] = {sub4(L[1], L[0]), sub4(L[2], L[1]), sub4(L[3], L[2])};
  double h = u1 - u0;
  d4 H00 = hblossom_d(D, u0, u0), H01 = hblossom_d(D, u0, u1), H11 = hblossom_d(D, u1, u1);
  d4 H0u = hblossom_d(D, 0.0, u0);
  LeafD q;
  q.p = fma4(u0, add4(add4(D[0], H0u), H00), L[0]);
  q.t0 = mul4(h, H00);
  q.t1 = mul4(h, H11);
  q.d = mul4(h, add4(add4(H00, H01), H11));
  return q;
}

__device__ __forceinline__ double cross_n2_d(d4 a, d4 b) {
  double cx = a.y * b.z - a.z * b.y, cy = a.z * b.x - a.x * b.z, cz = a.x * b.y - a.y * b.x;
  return cx * cx + cy * cy + cz * cz;
}

// Unit ray x leaf cylinder in FP64 (App. A), entry c0 of the infinite cylinder.
__device__ __forceinline__ bool cylinder_d(const LeafD& c, double& c0) {
  double dd = c.d.x * c.d.x + c.d.y * c.d.y + c.d.z * c.d.z;
  double m2 = fmax(cross_n2_d(c.t0, c.d), cross_n2_d(c.t1, c.d));
  double maxr = c.p.w + fmax(fmax(0.0, c.t0.w), fmax(c.d.w, c.d.w - c.t1.w));
  double R = sqrt(m2 / dd) + maxr;
  double g = c.d.x * c.d.x + c.d.y * c.d.y;
  if (!(g > 0.0)) return false;
  double h = 1.0 / g;
  double dxy = c.d.x * c.p.y - c.d.y * c.p.x;
  double e = R * R - dxy * dxy * h;
  if (!(e >= 0.0)) return false;
  double tc = c.p.z - c.d.z * (c.d.x * c.p.x + c.d.y * c.p.y) * h;
  c0 = tc - sqrt(e * (c.d.z * c.d.z + g) * h);
  return true;
}

// Finalisation (a7, lst:calc_intersection P:1546-1587 with F6, F8).  Re-solves the accepted
// leaf in FP64 from the input arrays; for lateral hits walks to the neighbouring leaf whose
// own slab contains the FP64 entry point (the FP32 leaf index can be a few leaves off at
// D >= 18 because leaves are then narrower than FP32 resolution).
__device__ __noinline__ void finalize(const float4 ray0, const float4 ray1, const float4 P0,
                                      const float4 P1, const float4 P2, const float4 P3,
                                      uint32_t start, int depth, uint32_t kind, float s32,
                                      float& t_out, float& u_out, uint32_t& n_out,
                                      bool& hit) {
  Frame F;
  make_frame(ray0, ray1, P0, P3, F);
  d4 L[4] = {to_local(F, P0), to_local(F, P1), to_local(F, P2), to_local(F, P3)};
  const int sh = FIBER_MAX_DEPTH - depth;
  const int64_t nleaf = (int64_t)1 << depth;
  int64_t k = (int64_t)(start >> sh);
  const double inv = 1.0 / (double)nleaf;
  double s = (double)s32, u = 0.0;
  d3 n = mk3(0, 0, 0);
  bool world_normal = false;
  if (kind == FIBER_KIND_CAP0 || kind == FIBER_KIND_CAP1) {
    // entry through a global cap plane: the plane of lst:calc_t_interval at u = 0 or 1
    d4 q = kind == FIBER_KIND_CAP0 ? L[0] : L[3];
    d4 nn = kind == FIBER_KIND_CAP0 ? sub4(L[1], L[0]) : sub4(L[3], L[2]);
    if (nn.z != 0.0) s = (q.x * nn.x + q.y * nn.y + q.z * nn.z) / nn.z;
    u = kind == FIBER_KIND_CAP0 ? 0.0 : 1.0;
    // cap normal in world space
    float4 a = kind == FIBER_KIND_CAP0 ? P0 : P3, b = kind == FIBER_KIND_CAP0 ? P1 : P2;
    n = mk3((double)a.x - b.x, (double)a.y - b.y, (double)a.z - b.z);
    world_normal = true;
  } else {
    LeafD q = leaf_d(L, k * inv, (k + 1) * inv);
    if (kind == FIBER_KIND_LATERAL) {
      double c0;
      if (cylinder_d(q, c0)) {
        s = c0;
        int dir = 0;
        for (int it = 0; it < 64; ++it) {
          // side of the entry point w.r.t. the leaf's own start / end planes
          double z0 = s - q.p.z;
          double side0 = -q.p.x * q.t0.x - q.p.y * q.t0.y + z0 * q.t0.z;
          double z1 = s - (q.p.z + q.d.z);
          double side1 = -(q.p.x + q.d.x) * q.t1.x - (q.p.y + q.d.y) * q.t1.y + z1 * q.t1.z;
          int step = 0;
          if (side0 < 0.0 && k > 0 && dir <= 0) step = -1;
          else if (side1 > 0.0 && k < nleaf - 1 && dir >= 0) step = +1;
          if (step == 0) break;
          LeafD qn = leaf_d(L, (k + step) * inv, (k + step + 1) * inv);
          double cn;
          if (!cylinder_d(qn, cn)) break;
          k += step;
          dir = step;
          q = qn;
          s = cn;
        }
      }
    }
    // u by projection onto the leaf chord, normal from the axis point (F8)
    double dd = q.d.x * q.d.x + q.d.y * q.d.y + q.d.z * q.d.z;
    double ul = ((0.0 - q.p.x) * q.d.x + (0.0 - q.p.y) * q.d.y + (s - q.p.z) * q.d.z) / dd;
    ul = fmin(1.0, fmax(0.0, ul));
    u = (k + ul) * inv;
    n = mk3(-(q.p.x + ul * q.d.x), -(q.p.y + ul * q.d.y), s - (q.p.z + ul * q.d.z));
  }
  double t = (F.ts + s) / F.lw;
  if (!world_normal) {
    n = mk3(n.x * F.b1.x + n.y * F.b2.x + n.z * F.w.x, n.x * F.b1.y + n.y * F.b2.y + n.z * F.w.y,
            n.x * F.b1.z + n.y * F.b2.z + n.z * F.w.z);
  }
  hit = t < (double)ray0.w;
  t_out = hit ? (float)t : INFINITY;
  u_out = hit ? (float)u : 0.0f;
  n_out = hit ? encode_oct(n.x, n.y, n.z) : 0u;
}

// ------------------------------------------------------------------------------------
// the per-pair traversal
// ------------------------------------------------------------------------------------
template <bool kNearest>
__global__ void __launch_bounds__(256) intersect_kernel(
    const float4* __restrict__ rays, int64_t n_rays, const float4* __restrict__ sp0,
    const float4* __restrict__ sp1, const float4* __restrict__ sp2, const float4* __restrict__ sp3,
    const uint32_t* __restrict__ sflags, int64_t n_segs, const uint2* __restrict__ pairs,
    int64_t n_pairs, int depth, float4* __restrict__ hits,
    unsigned long long* __restrict__ nearest) {
  const uint32_t min_size = 1u << (FIBER_MAX_DEPTH - depth);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pairs;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint2 pr = __ldg(&pairs[i]);
    uint32_t flags = 0;
    float t_out = INFINITY, u_out = 0.0f;
    uint32_t n_out = 0;
    if ((int64_t)pr.x >= n_rays || (int64_t)pr.y >= n_segs) {
      flags = FIBER_BAD_INPUT;
    } else {
      const float4 ray0 = __ldg(&rays[2 * (int64_t)pr.x]);
      const float4 ray1 = __ldg(&rays[2 * (int64_t)pr.x + 1]);
      const float4 P0 = __ldg(&sp0[pr.y]), P1 = __ldg(&sp1[pr.y]);
      const float4 P2 = __ldg(&sp2[pr.y]), P3 = __ldg(&sp3[pr.y]);
      if (__ldg(&sflags[pr.y]) != 0u) flags |= FIBER_BAD_SEGMENT;
      // ---- a2: FP64 setup: frame, transform (lst:transform_curve P:1482-1512), rounding
      Frame F;
      bool ok = make_frame(ray0, ray1, P0, P3, F);
      if (!ok) {
        flags |= FIBER_BAD_INPUT;
      } else {
        d4 L0 = to_local(F, P0), L1 = to_local(F, P1), L2 = to_local(F, P2), L3 = to_local(F, P3);
        Hodo hc;
        hc.L0 = to_f4(L0);
        hc.D0 = to_f4(sub4(L1, L0));
        hc.D1 = to_f4(sub4(L2, L1));
        hc.D2 = to_f4(sub4(L3, L2));
        Delta cur;  // conversion {p0,p1,p2,p3} -> {p,d,t0,t1} (3.1 P:372-375)
        cur.p = hc.L0;
        cur.d = to_f4(sub4(L3, L0));
        cur.t0 = hc.D0;
        cur.t1 = hc.D2;
        // ray interval [0, tmax) in local distance units s = t |d| - ts
        const float lo0 = (float)(-F.ts);
        const float hi0 = (float)((double)ray0.w * F.lw - F.ts);
        float tmin, tmax;
        uint32_t tag;
        slab(cur, lo0, hi0, true, true, tmin, tmax, tag);
        uint32_t bits = 0, size = 1u << FIBER_MAX_DEPTH, start = 0;
        uint32_t tests = 0, backtracks = 0;
        bool found = false;
        float c0 = 0.0f, c1 = 0.0f;
        // ---- a3-a6: the stackless loop
        while (true) {
          ++tests;
          bool pass = cylinder(cur, c0, c1);
          // pruning test P:1618 with F1 (empty interval) and F5 (explicit miss)
          pass = pass && (c1 >= tmin) && (c0 <= tmax) && (tmin <= tmax);
          if (pass) {
            if (size <= min_size) {  // leaf: first hit terminates
              found = true;
              break;
            }
            bool right, both;
            descend(cur, c0, c1, tmin, tmax, tag, right, both);
            // go_down (lst:bitstring_manipulation P:1516-1528)
            size >>= 1;
            if (both) bits |= size;
            if (right) start |= size;
          } else {
            if (bits == 0u) break;  // done
            ++backtracks;
            // jump_up: ctz of the pending bit string
            size = bits & (0u - bits);
            start ^= size;
            bits ^= size;
            start &= ~(size - 1u);
            float u0, u1;
            get_interval(start, size, u0, u1);
            recompute(hc, u0, u1, cur);
            slab(cur, lo0, hi0, start == 0u, start + size == (1u << FIBER_MAX_DEPTH), tmin, tmax,
                 tag);
          }
        }
        if (found) {
          // F2: entry into the cropped cylinder; F6: kind from the binding constraint
          float sstar = fmaxf(c0, tmin);
          uint32_t kind = FIBER_KIND_LATERAL;
          bool inside = false;
          if (!(c0 >= tmin)) {
            if (tag == TAG_ORIGIN) inside = true;
            else if (tag == TAG_START && start == 0u) kind = FIBER_KIND_CAP0;
            else if (tag == TAG_END && start + size == (1u << FIBER_MAX_DEPTH)) kind = FIBER_KIND_CAP1;
            else kind = FIBER_KIND_WEDGE;
          }
          bool hit = sstar < tmax;
          if (inside) {
            kind = FIBER_KIND_WEDGE;  // finalise like a crop-plane entry at s = -ts
            sstar = lo0;
          }
          if (hit) {
            finalize(ray0, ray1, P0, P1, P2, P3, start, depth, kind, sstar, t_out, u_out, n_out, hit);
            if (inside) {
              t_out = hit ? 0.0f : t_out;
              kind = FIBER_KIND_LATERAL;
            }
          }
          if (hit) flags |= FIBER_HIT | (kind << FIBER_KIND_SHIFT) | (inside ? FIBER_INSIDE : 0u);
        }
        flags |= (min(backtracks, 255u) << 8) | (min(tests, 65535u) << 16);
      }
    }
    if (hits) hits[i] = make_float4(t_out, u_out, __uint_as_float(n_out), __uint_as_float(flags));
    if (kNearest && (flags & FIBER_HIT)) {
      unsigned long long key =
          ((unsigned long long)__float_as_uint(t_out) << 32) | (unsigned long long)(uint32_t)i;
      atomicMin(&nearest[pr.x], key);
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

static int launch_intersect(const fiber_ray* rays, int64_t n_rays, const fiber_segments* segs,
                            const fiber_pair* pairs, int64_t n_pairs, int max_depth,
                            fiber_hit* hits, uint64_t* nearest, void* stream) {
  if (n_rays < 0 || n_pairs < 0 || n_rays >= ((int64_t)1 << 32) ||
      n_pairs >= ((int64_t)1 << 32) || max_depth < 0 || max_depth > FIBER_MAX_DEPTH || !segs)
    return set_error(FIBER_EINVAL, "fiber_intersect: bad size or depth");
  if (n_pairs > 0 && (!rays || !pairs || (!hits && !nearest) || !segs->p0 || !segs->p1 ||
                      !segs->p2 || !segs->p3 || !segs->flags))
    return set_error(FIBER_EINVAL, "fiber_intersect: NULL pointer");
  int rc = check_device();
  if (rc != FIBER_OK) return rc;
  if (n_pairs == 0) return FIBER_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (n_pairs + 255) / 256;
  int64_t cap = (int64_t)sms * 8;
  if (blocks > cap) blocks = cap;
  if (nearest) {
    intersect_kernel<true><<<(unsigned)blocks, 256, 0, st>>>(
        (const float4*)rays, n_rays, (const float4*)segs->p0, (const float4*)segs->p1,
        (const float4*)segs->p2, (const float4*)segs->p3, segs->flags, segs->n,
        (const uint2*)pairs, n_pairs, max_depth, (float4*)hits, (unsigned long long*)nearest);
  } else {
    intersect_kernel<false><<<(unsigned)blocks, 256, 0, st>>>(
        (const float4*)rays, n_rays, (const float4*)segs->p0, (const float4*)segs->p1,
        (const float4*)segs->p2, (const float4*)segs->p3, segs->flags, segs->n,
        (const uint2*)pairs, n_pairs, max_depth, (float4*)hits, nullptr);
  }
  return check_launch("fiber_intersect");
}

extern "C" int fiber_intersect(const fiber_ray* rays, int64_t n_rays, const fiber_segments* segs,
                               const fiber_pair* pairs, int64_t n_pairs, int max_depth,
                               fiber_hit* hits, void* cuda_stream) {
  if (n_pairs > 0 && !hits) return set_error(FIBER_EINVAL, "fiber_intersect: NULL hits");
  return launch_intersect(rays, n_rays, segs, pairs, n_pairs, max_depth, hits, nullptr,
                          cuda_stream);
}

extern "C" int fiber_intersect_nearest(const fiber_ray* rays, int64_t n_rays,
                                       const fiber_segments* segs, const fiber_pair* pairs,
                                       int64_t n_pairs, int max_depth, fiber_hit* hits,
                                       uint64_t* nearest, void* cuda_stream) {
  if (n_pairs > 0 && !nearest) return set_error(FIBER_EINVAL, "fiber_intersect_nearest: NULL nearest");
  return launch_intersect(rays, n_rays, segs, pairs, n_pairs, max_depth, hits, nearest,
                          cuda_stream);
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

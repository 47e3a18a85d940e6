// presplit.cu -- the input gatekeeper's pre-splitting and u remapping (
// 3.4 P:609-703: invalid curves and thick / cusp regions "must be subdivided beforehand").
// One thread per source segment runs the midpoint bisection depth-first (FP64, gatekeeper.cuh)
// twice: once to count its pieces, once to write them at the scanned offsets.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "fiber.h"
#include "fiber_internal.h"
#include "gatekeeper.cuh"

namespace {

constexpr int kMaxLevel = 16;

__device__ void load_cubic(const float* ctrl, const float* radii, int64_t s, double P[4][4]) {
  for (int i = 0; i < 4; ++i) {
    for (int k = 0; k < 3; ++k) P[i][k] = ctrl[12 * s + 3 * i + k];
    P[i][3] = radii[4 * s + i];
  }
}

// Depth-first bisection of [0, 1]; calls emit(u0, u1, valid, Q) for every piece in order.
template <class Emit>
__device__ void bisect(const double P[4][4], int max_level, bool parametric, Emit emit) {
  // explicit stack of (level, index): the interval is [index, index + 1] * 2^-level
  int lv[kMaxLevel + 2];
  uint32_t ix[kMaxLevel + 2];
  int top = 0;
  lv[0] = 0;
  ix[0] = 0;
  while (top >= 0) {
    const int level = lv[top];
    const uint32_t idx = ix[top];
    --top;
    const double h = ldexp(1.0, -level);
    const double u0 = idx * h, u1 = (idx + 1) * h;
    double Q[4][4];
    fibergk::subcurve(P, u0, u1, Q);
    const bool ok = fibergk::piece_valid(Q, parametric);
    if (ok || level >= max_level) {
      emit(u0, u1, ok, Q);
      continue;
    }
    lv[++top] = level + 1;  // right half below the left one: the left is taken first
    ix[top] = 2 * idx + 1;
    lv[++top] = level + 1;
    ix[top] = 2 * idx;
  }
}

__global__ void __launch_bounds__(128) presplit_count_kernel(const float* __restrict__ ctrl,
                                                            const float* __restrict__ radii,
                                                            int64_t n, int max_level,
                                                            int parametric,
                                                            uint32_t* __restrict__ counts) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    double P[4][4];
    load_cubic(ctrl, radii, s, P);
    uint32_t c = 0;
    bisect(P, max_level, parametric != 0, [&](double, double, bool, const double (*)[4]) { ++c; });
    counts[s + 1] = c;
  }
}

// In-place exclusive scan of counts[1..n] into offsets[0..n] (offsets[0] = 0), one block:
// every thread owns a contiguous chunk, the chunk sums are scanned in shared memory.
__global__ void __launch_bounds__(1024) scan_offsets_kernel(uint32_t* __restrict__ off, int64_t n) {
  __shared__ uint32_t part[1024];
  const int64_t chunk = (n + blockDim.x - 1) / blockDim.x;
  const int64_t b = 1 + threadIdx.x * chunk, e = min(n + 1, b + chunk);
  uint32_t sum = 0;
  for (int64_t i = b; i < e; ++i) sum += off[i];
  part[threadIdx.x] = sum;
  __syncthreads();
  for (int d = 1; d < (int)blockDim.x; d <<= 1) {  // Hillis-Steele inclusive scan
    uint32_t v = threadIdx.x >= (unsigned)d ? part[threadIdx.x - d] : 0u;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  uint32_t run = threadIdx.x ? part[threadIdx.x - 1] : 0u;
  for (int64_t i = b; i < e; ++i) {
    run += off[i];
    off[i] = run;
  }
  if (threadIdx.x == 0) off[0] = 0;
}

__global__ void __launch_bounds__(128) presplit_write_kernel(
    const float* __restrict__ ctrl, const float* __restrict__ radii, int64_t n, int max_level,
    int parametric, const uint32_t* __restrict__ off, float* __restrict__ out_ctrl,
    float* __restrict__ out_radii, uint32_t* __restrict__ out_src, float* __restrict__ out_u,
    uint32_t* __restrict__ out_valid) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    double P[4][4];
    load_cubic(ctrl, radii, s, P);
    uint32_t k = off[s];
    bisect(P, max_level, parametric != 0, [&](double u0, double u1, bool ok, const double (*Q)[4]) {
      for (int i = 0; i < 4; ++i) {
        for (int c = 0; c < 3; ++c) out_ctrl[12 * (int64_t)k + 3 * i + c] = (float)Q[i][c];
        out_radii[4 * (int64_t)k + i] = (float)Q[i][3];
      }
      out_src[k] = (uint32_t)s;
      out_u[2 * (int64_t)k] = (float)u0;
      out_u[2 * (int64_t)k + 1] = (float)u1;
      out_valid[k] = ok ? 1u : 0u;
      ++k;
    });
  }
}

__global__ void remap_u_kernel(float4* __restrict__ hits, const uint2* __restrict__ pairs,
                               int64_t n_pairs, const float2* __restrict__ piece_u,
                               int64_t n_pieces) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pairs;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 h = hits[i];
    uint32_t f = __float_as_uint(h.w);
    const uint32_t k = pairs[i].y;
    if (!(f & FIBER_HIT) || (int64_t)k >= n_pieces) continue;
    const float2 pu = piece_u[k];
    h.y = fmaf(h.y, pu.y - pu.x, pu.x);
    const uint32_t kind = (f & FIBER_KIND_MASK) >> FIBER_KIND_SHIFT;
    if ((kind == FIBER_KIND_CAP0 && pu.x > 0.0f) || (kind == FIBER_KIND_CAP1 && pu.y < 1.0f))
      f = (f & ~FIBER_KIND_MASK) | (FIBER_KIND_WEDGE << FIBER_KIND_SHIFT);
    h.w = __uint_as_float(f);
    hits[i] = h;
  }
}

int grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  return (int)(b > 148 * 32 ? 148 * 32 : (b < 1 ? 1 : b));
}

}  // namespace

extern "C" int fiber_presplit_count(const float* ctrl_pts, const float* radii, int64_t n,
                                    int max_level, int parametric, uint32_t* offsets,
                                    void* cuda_stream) {
  if (n < 0 || n >= ((int64_t)1 << 32) || max_level < 0 || max_level > kMaxLevel ||
      (n > 0 && (!ctrl_pts || !radii)) || !offsets)
    return set_error(FIBER_EINVAL, "fiber_presplit_count: bad arguments");
  int rc = check_device();
  if (rc != FIBER_OK) return rc;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (n > 0) {
    presplit_count_kernel<<<grid_for(n, 128), 128, 0, st>>>(ctrl_pts, radii, n, max_level,
                                                            parametric, offsets);
    rc = check_launch("fiber_presplit_count");
    if (rc != FIBER_OK) return rc;
  }
  scan_offsets_kernel<<<1, 1024, 0, st>>>(offsets, n);
  return check_launch("fiber_presplit_count (scan)");
}

extern "C" int fiber_presplit_write(const float* ctrl_pts, const float* radii, int64_t n,
                                    int max_level, int parametric, const uint32_t* offsets,
                                    float* out_ctrl, float* out_radii, uint32_t* out_src,
                                    float* out_u, uint32_t* out_valid, void* cuda_stream) {
  if (n < 0 || n >= ((int64_t)1 << 32) || max_level < 0 || max_level > kMaxLevel ||
      (n > 0 && (!ctrl_pts || !radii || !offsets || !out_ctrl || !out_radii || !out_src ||
                 !out_u || !out_valid)))
    return set_error(FIBER_EINVAL, "fiber_presplit_write: bad arguments");
  int rc = check_device();
  if (rc != FIBER_OK) return rc;
  if (n == 0) return FIBER_OK;
  presplit_write_kernel<<<grid_for(n, 128), 128, 0, (cudaStream_t)cuda_stream>>>(
      ctrl_pts, radii, n, max_level, parametric, offsets, out_ctrl, out_radii, out_src, out_u,
      out_valid);
  return check_launch("fiber_presplit_write");
}

extern "C" int fiber_remap_u(fiber_hit* hits, const fiber_pair* pairs, int64_t n_pairs,
                             const float* piece_u, int64_t n_pieces, void* cuda_stream) {
  if (n_pairs < 0 || n_pieces < 0 || (n_pairs > 0 && (!hits || !pairs || !piece_u)))
    return set_error(FIBER_EINVAL, "fiber_remap_u: bad arguments");
  int rc = check_device();
  if (rc != FIBER_OK) return rc;
  if (n_pairs == 0) return FIBER_OK;
  remap_u_kernel<<<grid_for(n_pairs, 256), 256, 0, (cudaStream_t)cuda_stream>>>(
      (float4*)hits, (const uint2*)pairs, n_pairs, (const float2*)piece_u, n_pieces);
  return check_launch("fiber_remap_u");
}

// scan.cuh -- device-wide exclusive prefix sum of uint32 (three phases: block sums, a
// single-block scan of the block sums, block scans plus the block prefix).  Used by the
// candidate generator (grid.cu) and the hit compaction (compact.cu).  In-place allowed.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace fiberscan {
namespace {  // internal linkage: every translation unit that includes this gets its own kernels

constexpr int kThreads = 256, kPer = 4, kTile = kThreads * kPer;  // 1024 elements per block

__device__ __forceinline__ uint32_t warp_incl(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += y;
  }
  return v;
}

// exclusive block scan of one value per thread; returns the block total in *total
__device__ __forceinline__ uint32_t block_excl(uint32_t v, uint32_t* total) {
  __shared__ uint32_t ws[kThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t inc = warp_incl(v);
  if (lane == 31) ws[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint32_t x = lane < kThreads / 32 ? ws[lane] : 0u;
    x = warp_incl(x);
    if (lane < kThreads / 32) ws[lane] = x;
  }
  __syncthreads();
  const uint32_t before = warp ? ws[warp - 1] : 0u;
  *total = ws[kThreads / 32 - 1];
  __syncthreads();
  return before + inc - v;
}

__global__ void __launch_bounds__(kThreads) block_sums(const uint32_t* __restrict__ in, int64_t n,
                                                      uint32_t* __restrict__ sums) {
  const int64_t base = (int64_t)blockIdx.x * kTile;
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int64_t i = base + k * kThreads + threadIdx.x;
    if (i < n) s += in[i];
  }
  uint32_t total;
  block_excl(s, &total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// single block: exclusive scan of sums[0..m) in place (chunked per thread)
__global__ void __launch_bounds__(1024) scan_sums(uint32_t* __restrict__ sums, int64_t m) {
  __shared__ uint32_t part[1024];
  const int64_t chunk = (m + blockDim.x - 1) / blockDim.x;
  const int64_t b = threadIdx.x * chunk, e = min(m, b + chunk);
  uint32_t s = 0;
  for (int64_t i = b; i < e; ++i) s += sums[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int d = 1; d < (int)blockDim.x; d <<= 1) {
    const uint32_t v = threadIdx.x >= (unsigned)d ? part[threadIdx.x - d] : 0u;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  uint32_t run = threadIdx.x ? part[threadIdx.x - 1] : 0u;
  for (int64_t i = b; i < e; ++i) {
    const uint32_t v = sums[i];
    sums[i] = run;
    run += v;
  }
}

__global__ void __launch_bounds__(kThreads) block_scan_add(const uint32_t* in, int64_t n,
                                                          const uint32_t* __restrict__ sums,
                                                          uint32_t* out) {
  // thread t owns elements base + t*kPer .. +kPer-1 (contiguous), so the scan is in order
  const int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kPer;
  uint32_t v[kPer], s = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    v[k] = base + k < n ? in[base + k] : 0u;
    s += v[k];
  }
  uint32_t total;
  uint32_t run = block_excl(s, &total) + sums[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    if (base + k < n) out[base + k] = run;
    run += v[k];
  }
}

// out[i] = sum of in[0..i) for i in [0, n); in == out allowed.  `sums` is scratch of
// ceil(n / 1024) uint32.  Returns the grid size used (0 if n == 0).
inline void exclusive_scan(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* sums,
                           cudaStream_t st) {
  if (n <= 0) return;
  const int64_t blocks = (n + kTile - 1) / kTile;
  block_sums<<<(unsigned)blocks, kThreads, 0, st>>>(in, n, sums);
  scan_sums<<<1, 1024, 0, st>>>(sums, blocks);
  block_scan_add<<<(unsigned)blocks, kThreads, 0, st>>>(in, n, sums, out);
}

inline int64_t scan_scratch(int64_t n) { return (n + kTile - 1) / kTile; }

}  // namespace
}  // namespace fiberscan

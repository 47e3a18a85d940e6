// compact.cu -- fiber_compact_hits: order-preserving stream compaction of hit records.
//
// A renderer consumes only the pairs that hit (the query returns the nearest
// intersection "or nothing"), so the records worth moving off the device are the hits.  Two
// passes over the records: per-tile hit counts, then each tile writes its hits at their
// global rank -- its offset summed from the counts before it (up to 4M records), else from a
// scan of the tile counts (scan.cuh) in between.  The result is deterministic: out[k] is the
// record of the k-th hit pair in pair order.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "fiber.h"
#include "fiber_internal.h"
#include "scan.cuh"

namespace fibercompact {

using fiberscan::kPer;
using fiberscan::kThreads;
using fiberscan::kTile;

// thread t of tile b owns records b*kTile + t*kPer .. +kPer-1 (contiguous, so ranks follow
// pair order)
__device__ __forceinline__ uint32_t tile_hits(const uint4* hits, int64_t n, int64_t base,
                                              uint32_t& mask) {
  uint32_t s = 0;
  mask = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    if (base + k < n && (__ldg(&hits[base + k].w) & FIBER_HIT)) {
      mask |= 1u << k;
      ++s;
    }
  }
  return s;
}

__global__ void __launch_bounds__(kThreads) count_kernel(const uint4* __restrict__ hits, int64_t n,
                                                        uint32_t* __restrict__ sums,
                                                        int64_t tiles) {
  const int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kPer;
  uint32_t mask;
  uint32_t total;
  fiberscan::block_excl(tile_hits(hits, n, base, mask), &total);
  if (threadIdx.x == 0) {
    sums[blockIdx.x] = total;
    if (blockIdx.x == 0) sums[tiles] = 0u;  // the scan's last element becomes the total
  }
}

__global__ void __launch_bounds__(kThreads) scatter_kernel(const uint4* __restrict__ hits, int64_t n,
                                                          const uint32_t* __restrict__ sums,
                                                          int64_t tiles, uint4* __restrict__ out,
                                                          uint32_t* __restrict__ idx,
                                                          uint32_t* __restrict__ count) {
  const int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kPer;
  uint32_t mask;
  uint32_t total;
  uint32_t run = fiberscan::block_excl(tile_hits(hits, n, base, mask), &total) + sums[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    if (mask & (1u << k)) {
      out[run] = __ldg(&hits[base + k]);
      if (idx) idx[run] = (uint32_t)(base + k);
      ++run;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *count = sums[tiles];
}

// Short inputs (up to kInlineTiles tiles, 4M records): the scatter forms its tile's offset
// itself -- a block reduction over the counts of the tiles before it (at most 16 KB, from L2)
// -- so the compaction is two kernels and no single-block scan between them.
constexpr int64_t kInlineTiles = 4096;
__global__ void __launch_bounds__(kThreads) scatter_inline_kernel(const uint4* __restrict__ hits,
                                                                 int64_t n,
                                                                 const uint32_t* __restrict__ sums,
                                                                 int64_t tiles,
                                                                 uint4* __restrict__ out,
                                                                 uint32_t* __restrict__ idx,
                                                                 uint32_t* __restrict__ count) {
  uint32_t part = 0, before;
  for (uint32_t t = threadIdx.x; t < blockIdx.x; t += kThreads) part += sums[t];
  fiberscan::block_excl(part, &before);
  const int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kPer;
  uint32_t mask;
  uint32_t total;
  uint32_t run = fiberscan::block_excl(tile_hits(hits, n, base, mask), &total) + before;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    if (mask & (1u << k)) {
      out[run] = __ldg(&hits[base + k]);
      if (idx) idx[run] = (uint32_t)(base + k);
      ++run;
    }
  }
  if (blockIdx.x == tiles - 1 && threadIdx.x == 0) *count = before + total;
}

}  // namespace fibercompact

extern "C" int fiber_compact_hits(const fiber_hit* hits, int64_t n, fiber_hit* out, uint32_t* idx,
                                  uint32_t* count, void* cuda_stream) {
  if (n < 0 || n >= ((int64_t)1 << 32) || !count || (n > 0 && (!hits || !out)))
    return set_error(FIBER_EINVAL, "fiber_compact_hits: bad size or NULL pointer");
  int rc = check_device();
  if (rc != FIBER_OK) return rc;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (n == 0) {
    if (cudaMemsetAsync(count, 0, sizeof(uint32_t), st) != cudaSuccess)
      return check_launch("fiber_compact_hits (memset)");
    return FIBER_OK;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool = scratch_pool(dev);
  const int64_t tiles = (n + fibercompact::kTile - 1) / fibercompact::kTile;
  uint32_t* sums = nullptr;
  cudaError_t e = pool ? cudaMallocFromPoolAsync((void**)&sums, (tiles + 1) * sizeof(uint32_t), pool, st)
                       : cudaErrorMemoryAllocation;
  if (e != cudaSuccess) {
    char buf[300];
    snprintf(buf, sizeof(buf), "fiber_compact_hits: scratch: %s", cudaGetErrorString(e));
    return set_error(FIBER_ECUDA, buf);
  }
  fibercompact::count_kernel<<<(unsigned)tiles, fibercompact::kThreads, 0, st>>>(
      (const uint4*)hits, n, sums, tiles);
  if (tiles <= fibercompact::kInlineTiles) {
    fibercompact::scatter_inline_kernel<<<(unsigned)tiles, fibercompact::kThreads, 0, st>>>(
        (const uint4*)hits, n, sums, tiles, (uint4*)out, idx, count);
  } else {
    fiberscan::scan_sums<<<1, 1024, 0, st>>>(sums, tiles + 1);
    fibercompact::scatter_kernel<<<(unsigned)tiles, fibercompact::kThreads, 0, st>>>(
        (const uint4*)hits, n, sums, tiles, (uint4*)out, idx, count);
  }
  rc = check_launch("fiber_compact_hits");
  cudaFreeAsync(sums, st);
  return rc;
}

// ------------------------------------------------------------------------------------
// fiber_nearest_records: the per-ray records of the nearest-hit epilogue (include/fiber.h)
// ------------------------------------------------------------------------------------
namespace fibercompact {
__global__ void records_kernel(const unsigned long long* __restrict__ nearest,
                               const uint4* __restrict__ hits, const uint2* __restrict__ pairs,
                               const int64_t* __restrict__ ray_ids, int64_t n,
                               uint4* __restrict__ out) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long key = nearest[__ldg(&ray_ids[j])];
    uint4 r = make_uint4(0x7f800000u, 0u, 0u, 0xffffffffu);  // +inf, no hit
    if (key != ~0ull) {
      const uint32_t i = (uint32_t)key;
      r = __ldg(&hits[i]);
      r.w = __ldg(&pairs[i]).y;
    }
    out[j] = r;
  }
}
}  // namespace fibercompact

extern "C" int fiber_nearest_records(const uint64_t* nearest, const fiber_hit* hits,
                                     const fiber_pair* pairs, const int64_t* ray_ids, int64_t n,
                                     fiber_hit* out, void* cuda_stream) {
  if (n < 0 || (n > 0 && (!nearest || !hits || !pairs || !ray_ids || !out)))
    return set_error(FIBER_EINVAL, "fiber_nearest_records: bad arguments");
  int rc = check_device();
  if (rc != FIBER_OK) return rc;
  if (n == 0) return FIBER_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  fibercompact::records_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)cuda_stream>>>(
      (const unsigned long long*)nearest, (const uint4*)hits, (const uint2*)pairs, ray_ids, n,
      (uint4*)out);
  return check_launch("fiber_nearest_records");
}

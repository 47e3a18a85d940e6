// Throughput of 64-bit REDG.MIN vs 32-bit REDG.MIN vs plain stores to random addresses of a
// 16 MB array (the C5 nearest-key epilogue: ~4.5M updates per 2^25-pair launch).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void red64(unsigned long long* a, uint32_t n_slots, uint32_t n_ops, uint32_t seed) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_ops; i += gridDim.x * blockDim.x) {
    uint32_t h = (i + seed) * 2654435761u;
    atomicMin(&a[h % n_slots], ((unsigned long long)h << 32) | i);
  }
}
__global__ void red32(unsigned* a, uint32_t n_slots, uint32_t n_ops, uint32_t seed) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_ops; i += gridDim.x * blockDim.x) {
    uint32_t h = (i + seed) * 2654435761u;
    atomicMin(&a[h % n_slots], h);
  }
}
__global__ void st64(unsigned long long* a, uint32_t n_slots, uint32_t n_ops, uint32_t seed) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_ops; i += gridDim.x * blockDim.x) {
    uint32_t h = (i + seed) * 2654435761u;
    a[h % n_slots] = ((unsigned long long)h << 32) | i;
  }
}
int main() {
  const uint32_t slots = 1u << 21, ops = 4500000;
  unsigned long long* a; cudaMalloc(&a, slots * 8ull);
  cudaMemset(a, 0xff, slots * 8ull);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int k = 0; k < 3; ++k) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (k == 0) red64<<<148 * 8, 256>>>(a, slots, ops, rep);
      if (k == 1) red32<<<148 * 8, 256>>>((unsigned*)a, slots * 2, ops, rep);
      if (k == 2) st64<<<148 * 8, 256>>>(a, slots, ops, rep);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("%s: %u ops in %.3f ms = %.2f G ops/s\n", k == 0 ? "red.min.64" : k == 1 ? "red.min.32" : "st.64", ops, ms, ops / ms / 1e6);
    }
  }
  return 0;
}

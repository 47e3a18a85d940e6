// Relative error of the MUFU FP64 seeds rcp.approx.ftz.f64 and rsqrt.approx.ftz.f64 over
// 2^24 log-uniform inputs in [2^-60, 2^60], and after one / two Newton steps.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__device__ double g_max[6];
__device__ __forceinline__ void amax(int k, double v) {
  unsigned long long* a = reinterpret_cast<unsigned long long*>(&g_max[k]);
  atomicMax(a, __double_as_longlong(fabs(v)));  // positive doubles order as integers
}
__global__ void k(int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned h = i * 2654435761u;
  double x = exp2(((h >> 8) / 16777216.0) * 120.0 - 60.0) * (1.0 + (h & 255) / 256.0);
  double r, y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e0 = fma(-x, r, 1.0);
  double r1 = fma(r, e0, r);
  double r2 = fma(r1, fma(-x, r1, 1.0), r1);
  double ref = 1.0 / x;
  amax(0, (r - ref) / ref); amax(1, (r1 - ref) / ref); amax(2, (r2 - ref) / ref);
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double sref = 1.0 / sqrt(x);
  double y1 = y * fma(-0.5 * x * y, y, 1.5);
  double y2 = y1 * fma(-0.5 * x * y1, y1, 1.5);
  amax(3, (y - sref) / sref); amax(4, (y1 - sref) / sref); amax(5, (y2 - sref) / sref);
}
int main() {
  int n = 1 << 24;
  k<<<n / 256, 256>>>(n);
  double h[6];
  cudaMemcpyFromSymbol(h, g_max, sizeof(h));
  const char* nm[] = {"rcp seed", "rcp 1 Newton", "rcp 2 Newton", "rsqrt seed", "rsqrt 1 Newton", "rsqrt 2 Newton"};
  for (int i = 0; i < 6; ++i) printf("%-16s max rel err %.3e (2^%.1f)\n", nm[i], h[i], log2(h[i]));
  return 0;
}

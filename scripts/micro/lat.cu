// Latency microbenchmark (one warp, dependent chains): DFMA, MUFU rcp/rsqrt f64 seeds,
// F2F f32<->f64, FFMA, FFMA2.  Prints cycles per dependent operation.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int N = 4096;
__global__ void k(double* out, float* outf, long long* cyc, double x0, float f0) {
  double x = x0; float f = f0;
  long long t0, t1;
#define RUN(ID, BODY) t0 = clock64(); for (int i = 0; i < N; ++i) { BODY; } t1 = clock64(); cyc[ID] = t1 - t0;
  RUN(0, x = fma(x, 0.999999, 1e-9))
  RUN(1, asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(x)))
  RUN(2, asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(x)))
  RUN(3, { float g = (float)x; x = (double)g; })
  RUN(4, f = fmaf(f, 0.9999f, 1e-7f))
  RUN(5, asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(f)))
  RUN(6, asm volatile("sqrt.approx.ftz.f32 %0, %0;" : "+f"(f)))
  RUN(7, { float2 v = __ffma2_rn(make_float2(f, f), make_float2(0.9999f, 0.9998f), make_float2(1e-7f, 1e-7f)); f = v.x + 0.0f * v.y; })
  RUN(8, x = x * 1.0000001 + 0.0)
  out[threadIdx.x] = x; outf[threadIdx.x] = f;
}
int main() {
  double* o; float* of; long long* c; long long h[16];
  cudaMalloc(&o, 1024 * 8); cudaMalloc(&of, 1024 * 4); cudaMalloc(&c, 16 * 8);
  for (int rep = 0; rep < 2; ++rep) {
    k<<<1, 32>>>(o, of, c, 1.5, 1.5f);
    cudaMemcpy(h, c, 16 * 8, cudaMemcpyDeviceToHost);
  }
  const char* names[] = {"DFMA", "MUFU.RCP64H", "MUFU.RSQ64H", "F2F f64->f32->f64 (2 ops)", "FFMA",
                         "MUFU.RCP f32", "MUFU.SQRT f32", "FFMA2 + FFMA", "DMUL+DADD"};
  for (int i = 0; i < 9; ++i) printf("%-28s %.1f cycles/iter\n", names[i], (double)h[i] / N);
  return 0;
}

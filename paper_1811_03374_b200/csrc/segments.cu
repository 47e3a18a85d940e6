// segments.cu -- K1: segment preprocessing.  One thread per segment: pack
// (ctrl_pts[n][4][3], radii[n][4]) into four float4 SoA planes (x, y, z, r) and validate
// the segment against the paper's preconditions (3.4).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "fiber.h"
#include "fiber_internal.h"
#include "gatekeeper.cuh"

namespace {

// The thick-fiber / cusp test at both ends (gatekeeper.cuh).
__device__ uint32_t thick_flags(const double P[4][3], const float r[4]) {
  double Q[4][4];
  for (int i = 0; i < 4; ++i) {
    for (int k = 0; k < 3; ++k) Q[i][k] = P[i][k];
    Q[i][3] = r[i];
  }
  uint32_t f = 0;
  if (fibergk::end_crossed(Q, 0, false) || fibergk::end_crossed(Q, 1, false)) {
    f |= FIBER_SEG_THICK;
    // r(u) <= r_bar: the exact surface can only cross where the r_bar surface does
    if (fibergk::end_crossed(Q, 0, true) || fibergk::end_crossed(Q, 1, true))
      f |= FIBER_SEG_THICK_PARAM;
  }
  return f;
}

__global__ void __launch_bounds__(256) build_segments_kernel(
    const float* __restrict__ ctrl, const float* __restrict__ radii, int64_t n,
    float4* __restrict__ p0, float4* __restrict__ p1, float4* __restrict__ p2,
    float4* __restrict__ p3, uint32_t* __restrict__ flags) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    double P[4][3];
    float r[4];
    uint32_t f = 0;
    for (int i = 0; i < 4; ++i) {
      r[i] = radii[4 * s + i];
      for (int k = 0; k < 3; ++k) {
        float v = ctrl[12 * s + 3 * i + k];
        if (!isfinite(v)) f |= FIBER_SEG_NONFINITE;
        P[i][k] = v;
      }
      if (!isfinite(r[i])) f |= FIBER_SEG_NONFINITE;
      if (r[i] < 0.0f) f |= FIBER_SEG_NEG_RADIUS;
    }
    auto dotd = [&](int a, int b, int c, int d) {  // <P_a - P_b, P_c - P_d>
      double acc = 0.0;
      for (int k = 0; k < 3; ++k) acc += (P[a][k] - P[b][k]) * (P[c][k] - P[d][k]);
      return acc;
    };
    // the five inequalities of P:616-620 (App. B eqs)
    if (dotd(2, 0, 1, 0) < 0.0) f |= FIBER_SEG_CONSTRAINT(0);
    if (dotd(3, 1, 1, 0) < 0.0) f |= FIBER_SEG_CONSTRAINT(1);
    if (dotd(3, 1, 3, 2) < 0.0) f |= FIBER_SEG_CONSTRAINT(2);
    if (dotd(2, 0, 3, 2) < 0.0) f |= FIBER_SEG_CONSTRAINT(3);
    if (dotd(2, 0, 3, 1) < 0.0) f |= FIBER_SEG_CONSTRAINT(4);
    // degenerate chord or end tangent: the cropping plane normal is undefined
    double dd = dotd(3, 0, 3, 0), a0 = dotd(1, 0, 1, 0), a1 = dotd(3, 2, 3, 2);
    if (!(dd > 0.0) || a0 <= 1e-12 * dd || a1 <= 1e-12 * dd) f |= FIBER_SEG_DEGENERATE;
    if (!(f & (FIBER_SEG_NONFINITE | FIBER_SEG_DEGENERATE))) f |= thick_flags(P, r);
    p0[s] = make_float4((float)P[0][0], (float)P[0][1], (float)P[0][2], r[0]);
    p1[s] = make_float4((float)P[1][0], (float)P[1][1], (float)P[1][2], r[1]);
    p2[s] = make_float4((float)P[2][0], (float)P[2][1], (float)P[2][2], r[2]);
    p3[s] = make_float4((float)P[3][0], (float)P[3][1], (float)P[3][2], r[3]);
    flags[s] = f;
  }
}

// Quadratic segments: validate (App. B.1) and store unrounded; the kernels elevate.
__global__ void __launch_bounds__(256) build_quadratic_kernel(
    const float* __restrict__ ctrl, const float* __restrict__ radii, int64_t n,
    float4* __restrict__ p0, float4* __restrict__ p1, float4* __restrict__ p2,
    float4* __restrict__ p3, uint32_t* __restrict__ flags) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    double Q[3][3];
    float r[3];
    uint32_t f = FIBER_SEG_QUADRATIC;
    for (int i = 0; i < 3; ++i) {
      r[i] = radii[3 * s + i];
      for (int k = 0; k < 3; ++k) {
        float v = ctrl[9 * s + 3 * i + k];
        if (!isfinite(v)) f |= FIBER_SEG_NONFINITE;
        Q[i][k] = v;
      }
      if (!isfinite(r[i])) f |= FIBER_SEG_NONFINITE;
      if (r[i] < 0.0f) f |= FIBER_SEG_NEG_RADIUS;
    }
    auto dotd = [&](int a, int b, int c, int d) {  // <Q_a - Q_b, Q_c - Q_d>
      double acc = 0.0;
      for (int k = 0; k < 3; ++k) acc += (Q[a][k] - Q[b][k]) * (Q[c][k] - Q[d][k]);
      return acc;
    };
    if (dotd(1, 0, 1, 2) > 0.0) f |= FIBER_SEG_QUAD_CONSTRAINT;  // eq. P:889
    double dd = dotd(2, 0, 2, 0), a0 = dotd(1, 0, 1, 0), a1 = dotd(2, 1, 2, 1);
    if (!(dd > 0.0) || a0 <= 1e-12 * dd || a1 <= 1e-12 * dd) f |= FIBER_SEG_DEGENERATE;
    if (!(f & (FIBER_SEG_NONFINITE | FIBER_SEG_DEGENERATE))) {
      // the thick-fiber test on the exact elevation
      double E[4][3];
      float re[4];
      for (int k = 0; k < 3; ++k) {
        E[0][k] = Q[0][k];
        E[1][k] = (Q[0][k] + 2.0 * Q[1][k]) / 3.0;
        E[2][k] = (2.0 * Q[1][k] + Q[2][k]) / 3.0;
        E[3][k] = Q[2][k];
      }
      re[0] = r[0];
      re[1] = (float)(((double)r[0] + 2.0 * r[1]) / 3.0);
      re[2] = (float)((2.0 * r[1] + (double)r[2]) / 3.0);
      re[3] = r[2];
      f |= thick_flags(E, re);
    }
    const float4 q1 = make_float4((float)Q[1][0], (float)Q[1][1], (float)Q[1][2], r[1]);
    p0[s] = make_float4((float)Q[0][0], (float)Q[0][1], (float)Q[0][2], r[0]);
    p1[s] = q1;
    p2[s] = q1;
    p3[s] = make_float4((float)Q[2][0], (float)Q[2][1], (float)Q[2][2], r[2]);
    flags[s] = f;
  }
}

}  // namespace

extern "C" int fiber_build_segments_quadratic(const float* ctrl_pts, const float* radii,
                                              int64_t n, fiber_segments* segs,
                                              void* cuda_stream) {
  if (n < 0 || n >= ((int64_t)1 << 32) || !segs || segs->n != n)
    return set_error(FIBER_EINVAL, "fiber_build_segments_quadratic: bad size or descriptor");
  if (n > 0 && (!ctrl_pts || !radii || !segs->p0 || !segs->p1 || !segs->p2 || !segs->p3 ||
                !segs->flags))
    return set_error(FIBER_EINVAL, "fiber_build_segments_quadratic: NULL pointer");
  int rc = check_device();
  if (rc != FIBER_OK) return rc;
  if (n == 0) return FIBER_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  build_quadratic_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)cuda_stream>>>(
      ctrl_pts, radii, n, (float4*)segs->p0, (float4*)segs->p1, (float4*)segs->p2,
      (float4*)segs->p3, segs->flags);
  return check_launch("fiber_build_segments_quadratic");
}

extern "C" int fiber_build_segments(const float* ctrl_pts, const float* radii, int64_t n,
                                    fiber_segments* segs, void* cuda_stream) {
  if (n < 0 || n >= ((int64_t)1 << 32) || !segs || segs->n != n)
    return set_error(FIBER_EINVAL, "fiber_build_segments: bad size or descriptor");
  if (n > 0 && (!ctrl_pts || !radii || !segs->p0 || !segs->p1 || !segs->p2 || !segs->p3 ||
                !segs->flags))
    return set_error(FIBER_EINVAL, "fiber_build_segments: NULL pointer");
  int rc = check_device();
  if (rc != FIBER_OK) return rc;
  if (n == 0) return FIBER_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  build_segments_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)cuda_stream>>>(
      ctrl_pts, radii, n, (float4*)segs->p0, (float4*)segs->p1, (float4*)segs->p2,
      (float4*)segs->p3, segs->flags);
  return check_launch("fiber_build_segments");
}

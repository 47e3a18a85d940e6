// gatekeeper.cuh -- the input gatekeeper's device arithmetic: the
// thick-fiber / cusp test of 3.4 as a certified polynomial sign test, and the
// sub-curve blossom used by pre-splitting.  FP64; used by K1 (segments.cu) and the
// pre-split kernels (presplit.cu).
//
// The test.  For the end plane through p3 with normal t1 = C'(1),
// the normal disc at u (centre C(u), normal T(u) = C'(u), radius r) reaches furthest across
// the plane at C(u) + r n^_u, n_u the Gram-Schmidt displacement of P:676-682, and
// <n^_u, t^1> = |T(u) x t1| / (|T(u)| |t1|).  The surface stays inside iff for all u
//     A(u) |T(u)| >= r(u) |X(u)|,   A(u) = <p3 - C(u), t1>,  X(u) = T(u) x t1.
// Both A and X vanish at u = 1; dividing by (1 - u) (exact in the Bernstein basis) gives
// A~ (degree 2) and X~ (degree 1), and the condition is A~(u) >= 0 and
//     F(u) = A~(u)^2 |T(u)|^2 - r(u)^2 |X~(u)|^2 >= 0,
// a polynomial of degree 8 for both the constant r_bar and the cubic r(u).
// (The paper solves a quartic by Ferrari's method; with the normalisation of
// n_u the condition is not quartic, so the sign of F is certified instead: Bernstein
// coefficients bound the polynomial on an interval (convex hull), and de Casteljau halving
// refines where the bound is inconclusive.)  The p0 end is the same test on the reversed
// curve.
#pragma once
#include <cstdint>

namespace fibergk {

// Polynomials in the Bernstein basis of fixed degree N on [0, 1] (degrees are template
// parameters, so the coefficient arrays live in registers and the loops unroll).
template <int N>
struct BP {
  double b[N + 1];
};

__host__ __device__ constexpr double binom(int n, int k) {
  double r = 1.0;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}

template <int M, int N>
__device__ __forceinline__ BP<M + N> bp_mul(const BP<M>& f, const BP<N>& g) {
  BP<M + N> r;
#pragma unroll
  for (int k = 0; k <= M + N; ++k) r.b[k] = 0.0;
#pragma unroll
  for (int i = 0; i <= M; ++i)
#pragma unroll
    for (int j = 0; j <= N; ++j) r.b[i + j] += (binom(M, i) * binom(N, j)) * f.b[i] * g.b[j];
#pragma unroll
  for (int k = 0; k <= M + N; ++k) r.b[k] *= 1.0 / binom(M + N, k);
  return r;
}

template <int N, int M>
__device__ __forceinline__ BP<M> bp_elevate(const BP<N>& f) {
  BP<M> r;
#pragma unroll
  for (int k = 0; k <= M; ++k) {
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i <= N; ++i)
      if (k - i >= 0 && k - i <= M - N) acc += (binom(N, i) * binom(M - N, k - i)) * f.b[i];
    r.b[k] = acc * (1.0 / binom(M, k));
  }
  return r;
}

// True iff f(u) < -tol for some u in [0, 1], certified by the convex hull of the Bernstein
// coefficients and de Casteljau halving (depth-first, explicit stack).  At the depth limit
// the midpoint value decides (the polynomial is then within rounding of a root).
template <int N>
__device__ __noinline__ bool bp_negative_somewhere(const BP<N> f0, double tol) {
  constexpr int kStack = 44, kMaxLevel = 40;
  BP<N> st[kStack];
  unsigned char lv[kStack];
  int top = 0;
  st[0] = f0;
  lv[0] = 0;
  while (top >= 0) {
    const BP<N> f = st[top];
    const int level = lv[top];
    --top;
    if (f.b[0] < -tol || f.b[N] < -tol) return true;  // an end value
    double mn = f.b[0];
#pragma unroll
    for (int k = 1; k <= N; ++k) mn = fmin(mn, f.b[k]);
    if (mn >= -tol) continue;  // hull above -tol on this interval
    double w[N + 1];
#pragma unroll
    for (int k = 0; k <= N; ++k) w[k] = f.b[k];
    BP<N> L, R;
    L.b[0] = w[0];
    R.b[N] = w[N];
#pragma unroll
    for (int r = 1; r <= N; ++r) {
#pragma unroll
      for (int k = 0; k <= N - r; ++k) w[k] = 0.5 * (w[k] + w[k + 1]);
      L.b[r] = w[0];
      R.b[N - r] = w[N - r];
    }
    if (level >= kMaxLevel || top + 2 >= kStack) {
      if (R.b[0] < -tol) return true;  // the midpoint value
      continue;
    }
    st[++top] = R;
    lv[top] = (unsigned char)(level + 1);
    st[++top] = L;  // left first
    lv[top] = (unsigned char)(level + 1);
  }
  return false;
}

// Control points P[4][4] = (x, y, z, r) of a cubic fiber.  Does the surface cross the plane
// of end `end` (1: through p3, normal p3 - p2; 0: through p0, normal p0 - p1)?  r = the
// largest radius control point (parametric = false) or the cubic radius (true).
__device__ inline bool end_crossed(const double Pin[4][4], int end, bool parametric) {
  double P[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k) P[i][k] = end ? Pin[i][k] : Pin[3 - i][k];
  // scale-free coordinates: relative to p0, divided by the chord length
  double ch = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) ch += (P[3][k] - P[0][k]) * (P[3][k] - P[0][k]);
  ch = sqrt(ch);
  if (!(ch > 0.0)) return true;
  const double is = 1.0 / ch;
  double Q[4][3];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) Q[i][k] = (P[i][k] - P[0][k]) * is;
  double T[3][3], t1[3];
#pragma unroll
  for (int j = 0; j < 3; ++j)
#pragma unroll
    for (int k = 0; k < 3; ++k) T[j][k] = 3.0 * (Q[j + 1][k] - Q[j][k]);
#pragma unroll
  for (int k = 0; k < 3; ++k) t1[k] = T[2][k];
  // A~ (degree 2): A_i = <Q3 - Q_i, t1>, A_3 = 0, divided by (1 - u): A~_i = A_i 3 / (3 - i)
  BP<2> At;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) a += (Q[3][k] - Q[i][k]) * t1[k];
    At.b[i] = a * 3.0 / (3.0 - i);
  }
  // |T|^2 (degree 4) and |X~|^2, X~ = (T x t1) / (1 - u) (degree 1): X_j 2 / (2 - j), X_2 = 0
  BP<4> T2;
  BP<2> X2;
#pragma unroll
  for (int k = 0; k <= 4; ++k) T2.b[k] = 0.0;
#pragma unroll
  for (int k = 0; k <= 2; ++k) X2.b[k] = 0.0;
  double Xt[2][3];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const double* a = T[j];
    Xt[j][0] = (a[1] * t1[2] - a[2] * t1[1]) * 2.0 / (2.0 - j);
    Xt[j][1] = (a[2] * t1[0] - a[0] * t1[2]) * 2.0 / (2.0 - j);
    Xt[j][2] = (a[0] * t1[1] - a[1] * t1[0]) * 2.0 / (2.0 - j);
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    BP<2> tc;
#pragma unroll
    for (int j = 0; j < 3; ++j) tc.b[j] = T[j][c];
    const BP<4> sq = bp_mul(tc, tc);
#pragma unroll
    for (int k = 0; k <= 4; ++k) T2.b[k] += sq.b[k];
    BP<1> xc;
    xc.b[0] = Xt[0][c];
    xc.b[1] = Xt[1][c];
    const BP<2> xs = bp_mul(xc, xc);
#pragma unroll
    for (int k = 0; k <= 2; ++k) X2.b[k] += xs.b[k];
  }
  BP<8> rhs;
  if (parametric) {
    BP<3> r;
#pragma unroll
    for (int i = 0; i < 4; ++i) r.b[i] = P[i][3] * is;
    rhs = bp_mul(bp_mul(r, r), X2);
  } else {
    const double rb = fmax(fmax(P[0][3], P[1][3]), fmax(P[2][3], P[3][3])) * is;
    const BP<8> x8 = bp_elevate<2, 8>(X2);
#pragma unroll
    for (int k = 0; k <= 8; ++k) rhs.b[k] = rb * rb * x8.b[k];
  }
  const BP<8> lhs = bp_mul(bp_mul(At, At), T2);
  BP<8> F;
  double sc = 0.0;
#pragma unroll
  for (int k = 0; k <= 8; ++k) {
    F.b[k] = lhs.b[k] - rhs.b[k];
    sc = fmax(sc, fmax(fabs(lhs.b[k]), fabs(rhs.b[k])));
  }
  const double sa = fmax(fabs(At.b[0]), fmax(fabs(At.b[1]), fabs(At.b[2])));
  return bp_negative_somewhere<2>(At, 1e-13 * sa) || bp_negative_somewhere<8>(F, 1e-13 * sc);
}

// The five cubic constraints hold (>= 0) on the positions of P.
__device__ inline bool constraints_ok(const double P[4][4]) {
  auto d = [&](int a, int b, int c, int e) {
    double acc = 0.0;
    for (int k = 0; k < 3; ++k) acc += (P[a][k] - P[b][k]) * (P[c][k] - P[e][k]);
    return acc;
  };
  return d(2, 0, 1, 0) >= 0.0 && d(3, 1, 1, 0) >= 0.0 && d(3, 1, 3, 2) >= 0.0 &&
         d(2, 0, 3, 2) >= 0.0 && d(2, 0, 3, 1) >= 0.0;
}

// Sub-curve on [u0, u1] by blossoming: Q_i = blossom(u0 x (3 - i), u1 x i) (de Casteljau),
// all four components.
__device__ inline void subcurve(const double P[4][4], double u0, double u1, double Q[4][4]) {
  for (int i = 0; i < 4; ++i) {
    double a[4][4];
    for (int j = 0; j < 4; ++j)
      for (int k = 0; k < 4; ++k) a[j][k] = P[j][k];
    for (int r = 1; r <= 3; ++r) {
      const double t = (r <= 3 - i) ? u0 : u1;
      for (int j = 0; j <= 3 - r; ++j)
        for (int k = 0; k < 4; ++k) a[j][k] = (1.0 - t) * a[j][k] + t * a[j + 1][k];
    }
    for (int k = 0; k < 4; ++k) Q[i][k] = a[0][k];
  }
}

// A piece passes the gatekeeper: constraints and neither end plane crossed.
__device__ inline bool piece_valid(const double Q[4][4], bool parametric) {
  return constraints_ok(Q) && !end_crossed(Q, 0, parametric) && !end_crossed(Q, 1, parametric);
}

}  // namespace fibergk

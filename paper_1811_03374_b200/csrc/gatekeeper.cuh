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

constexpr int kMaxDeg = 8;

struct BP {  // polynomial in the Bernstein basis of degree n on [0, 1]
  int n;
  double b[kMaxDeg + 1];
};

__device__ __forceinline__ double binom(int n, int k) {
  // n <= 8
  const double row[9][9] = {
      {1}, {1, 1}, {1, 2, 1}, {1, 3, 3, 1}, {1, 4, 6, 4, 1}, {1, 5, 10, 10, 5, 1},
      {1, 6, 15, 20, 15, 6, 1}, {1, 7, 21, 35, 35, 21, 7, 1}, {1, 8, 28, 56, 70, 56, 28, 8, 1}};
  return row[n][k];
}

__device__ inline BP bp_mul(const BP& f, const BP& g) {
  BP r;
  r.n = f.n + g.n;
  for (int k = 0; k <= r.n; ++k) r.b[k] = 0.0;
  for (int i = 0; i <= f.n; ++i)
    for (int j = 0; j <= g.n; ++j) r.b[i + j] += binom(f.n, i) * binom(g.n, j) * f.b[i] * g.b[j];
  for (int k = 0; k <= r.n; ++k) r.b[k] /= binom(r.n, k);
  return r;
}

__device__ inline BP bp_elevate(const BP& f, int N) {
  BP r;
  r.n = N;
  for (int k = 0; k <= N; ++k) {
    double acc = 0.0;
    for (int i = 0; i <= f.n; ++i)
      if (k - i >= 0 && k - i <= N - f.n) acc += binom(f.n, i) * binom(N - f.n, k - i) * f.b[i];
    r.b[k] = acc / binom(N, k);
  }
  return r;
}

__device__ inline BP bp_axpy(double a, const BP& f, const BP& g) {  // a f + g
  const int N = f.n > g.n ? f.n : g.n;
  const BP F = bp_elevate(f, N), G = bp_elevate(g, N);
  BP r;
  r.n = N;
  for (int k = 0; k <= N; ++k) r.b[k] = a * F.b[k] + G.b[k];
  return r;
}

// True iff f(u) < -tol for some u in [0, 1], certified by the convex hull of the Bernstein
// coefficients and de Casteljau halving (depth-first, explicit stack).  At the depth limit
// the midpoint value decides (the polynomial is then within rounding of a root).
__device__ inline bool bp_negative_somewhere(const BP& f0, double tol) {
  constexpr int kStack = 48, kMaxLevel = 40;
  BP st[kStack];
  int lv[kStack];
  int top = 0;
  st[0] = f0;
  lv[0] = 0;
  while (top >= 0) {
    const BP f = st[top];
    const int level = lv[top];
    --top;
    if (f.b[0] < -tol || f.b[f.n] < -tol) return true;  // an end value
    double mn = f.b[0];
    for (int k = 1; k <= f.n; ++k) mn = fmin(mn, f.b[k]);
    if (mn >= -tol) continue;  // hull above -tol on this interval
    if (level >= kMaxLevel || top + 2 >= kStack) {
      // value at the midpoint
      double w[kMaxDeg + 1];
      for (int k = 0; k <= f.n; ++k) w[k] = f.b[k];
      for (int r = 1; r <= f.n; ++r)
        for (int k = 0; k <= f.n - r; ++k) w[k] = 0.5 * (w[k] + w[k + 1]);
      if (w[0] < -tol) return true;
      continue;
    }
    // de Casteljau at 1/2: left = first column, right = last diagonal
    double w[kMaxDeg + 1];
    BP L, R;
    L.n = R.n = f.n;
    for (int k = 0; k <= f.n; ++k) w[k] = f.b[k];
    L.b[0] = w[0];
    R.b[f.n] = w[f.n];
    for (int r = 1; r <= f.n; ++r) {
      for (int k = 0; k <= f.n - r; ++k) w[k] = 0.5 * (w[k] + w[k + 1]);
      L.b[r] = w[0];
      R.b[f.n - r] = w[f.n - r];
    }
    st[++top] = R;
    lv[top] = level + 1;
    st[++top] = L;  // left first
    lv[top] = level + 1;
  }
  return false;
}

// Control points P[4][4] = (x, y, z, r) of a cubic fiber.  Does the surface cross the plane
// of end `end` (1: through p3, normal p3 - p2; 0: through p0, normal p0 - p1)?  r = the
// largest radius control point (parametric = false) or the cubic radius (true).
__device__ inline bool end_crossed(const double Pin[4][4], int end, bool parametric) {
  double P[4][4];
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < 4; ++k) P[i][k] = end ? Pin[i][k] : Pin[3 - i][k];
  // scale-free coordinates: relative to p0, divided by the chord length
  double ch = 0.0;
  for (int k = 0; k < 3; ++k) ch += (P[3][k] - P[0][k]) * (P[3][k] - P[0][k]);
  ch = sqrt(ch);
  if (!(ch > 0.0)) return true;
  const double is = 1.0 / ch;
  double Q[4][3];
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < 3; ++k) Q[i][k] = (P[i][k] - P[0][k]) * is;
  double T[3][3], t1[3];
  for (int j = 0; j < 3; ++j)
    for (int k = 0; k < 3; ++k) T[j][k] = 3.0 * (Q[j + 1][k] - Q[j][k]);
  for (int k = 0; k < 3; ++k) t1[k] = T[2][k];
  // A~ (degree 2): A_i = <Q3 - Q_i, t1>, A_3 = 0, divided by (1 - u): A~_i = A_i 3 / (3 - i)
  BP At;
  At.n = 2;
  for (int i = 0; i < 3; ++i) {
    double a = 0.0;
    for (int k = 0; k < 3; ++k) a += (Q[3][k] - Q[i][k]) * t1[k];
    At.b[i] = a * 3.0 / (3.0 - i);
  }
  // |T|^2 (degree 4) and X~ = (T x t1) / (1 - u) (degree 1): X_j 2 / (2 - j), X_2 = 0
  BP T2;
  T2.n = 4;
  for (int k = 0; k <= 4; ++k) T2.b[k] = 0.0;
  BP X2;
  X2.n = 2;
  for (int k = 0; k <= 2; ++k) X2.b[k] = 0.0;
  double Xt[2][3];
  for (int j = 0; j < 2; ++j) {
    const double* a = T[j];
    Xt[j][0] = (a[1] * t1[2] - a[2] * t1[1]) * 2.0 / (2.0 - j);
    Xt[j][1] = (a[2] * t1[0] - a[0] * t1[2]) * 2.0 / (2.0 - j);
    Xt[j][2] = (a[0] * t1[1] - a[1] * t1[0]) * 2.0 / (2.0 - j);
  }
  for (int c = 0; c < 3; ++c) {
    BP tc;
    tc.n = 2;
    for (int j = 0; j < 3; ++j) tc.b[j] = T[j][c];
    const BP sq = bp_mul(tc, tc);
    for (int k = 0; k <= 4; ++k) T2.b[k] += sq.b[k];
    BP xc;
    xc.n = 1;
    xc.b[0] = Xt[0][c];
    xc.b[1] = Xt[1][c];
    const BP xs = bp_mul(xc, xc);
    for (int k = 0; k <= 2; ++k) X2.b[k] += xs.b[k];
  }
  BP R2;
  if (parametric) {
    BP r;
    r.n = 3;
    for (int i = 0; i < 4; ++i) r.b[i] = P[i][3] * is;
    R2 = bp_mul(r, r);
  } else {
    const double rb = fmax(fmax(P[0][3], P[1][3]), fmax(P[2][3], P[3][3])) * is;
    R2.n = 0;
    R2.b[0] = rb * rb;
  }
  const BP lhs = bp_mul(bp_mul(At, At), T2);  // degree 8
  const BP rhs = bp_mul(R2, X2);               // degree 8 or 2
  const BP F = bp_axpy(-1.0, rhs, lhs);
  double sc = 0.0;
  for (int k = 0; k <= lhs.n; ++k) sc = fmax(sc, fabs(lhs.b[k]));
  for (int k = 0; k <= rhs.n; ++k) sc = fmax(sc, fabs(rhs.b[k]));
  double sa = 0.0;
  for (int k = 0; k <= 2; ++k) sa = fmax(sa, fabs(At.b[k]));
  return bp_negative_somewhere(At, 1e-13 * sa) || bp_negative_somewhere(F, 1e-13 * sc);
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

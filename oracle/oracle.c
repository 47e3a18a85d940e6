/*
 * oracle.c -- plain, slow, FP64 CPU oracle for the ray/fiber intersection of
 * Binder & Keller, "Fast, High Precision Ray/Fiber Intersection using Tight,
 * Disjoint Bounding Volumes" (arXiv 1811.03374).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_1811_03374_b200/) never links, imports or calls it, and
 * the two share no code, headers, tables or helpers.
 *
 * What it computes: the paper's algorithm
 * at subdivision depth D, written as a plain recursion in WORLD space with the
 * general formulas -- no ray frame, no (p,d,t0,t1) delta form, no bit string.
 * Every node's sub-curve is re-evaluated from the original control points.
 *
 *   PAPER.md citations (P:line):
 *   - Bernstein evaluation / (scaled) derivative       lst:eval_cubic_bezier P:1347-1364
 *   - node sub-curve from eval/eval_derivative          lst:recalculation
 *   - conservative radius: max inner-CP distance to the
 *     chord + max radius CP (convex hull)               P:488-495, lst:calc_radius P:1415-1425,
 *                                                       lst:distance-point-line P:1308-1328
 *   - cylinder = {x : dist(x, chord line) <= R}          App. A P:785-874 (the unit-ray
 *                                                       specialisation of this definition)
 *   - cropping planes through the end points, normal =
 *     end tangents                                      P:497-500, lst:calc_t_interval P:1459-1477
 *   - partition plane through the split point, normal =
 *     split tangent; near-first order; both-hit test;
 *     one-bound update                                  3.2 P:453-471, lst:subdivide_partition_and_update
 *                                                       P:1429-1456, fig:bounding_cylinder P:515-606
 *   - first leaf hit terminates                         P:357-359, 464-467, lst:algorithm
 *   - u by projection onto the leaf chord, cap normals,
 *     normal = hit - axis point                          lst:calc_intersection P:1546-1587
 *   - the five cubic constraints                        3.4 P:614-621 (App. B eqs)
 *
 *   Readings where the listings are silent or wrong (F1-F9):
 *   F1 an interval with lo > hi is empty (listing P:1618 passes it)
 *   F2 leaf hit t* = max(c0, lo), the entry into the CROPPED cylinder (P:1622 says t0)
 *   F3 a plane parallel to the ray is a half-space test: the ray is wholly valid or
 *      wholly invalid; near child = the side the ray lies on; no both; no bound update
 *   F4 ray parallel to the axis: the whole line if inside, else empty
 *   F5 a miss is an explicit empty interval, never a FLT_MAX sentinel
 *   F6 the hit kind comes from the binding constraint (global caps), not from u == 0/1
 *   F7 after backtracking the interval is the far node's own slab with the ray's t_max
 *   F8 the leaf axis is the leaf chord
 *   F9 near child = XOR of the two comparisons; the curve is in/out
 *
 * Grazing band: eps_sign = +1/-1 re-runs the same recursion
 * with every cylinder radius grown/shrunk by eps, the two GLOBAL cap planes (u = 0,
 * u = 1) moved outward/inward by eps, and every INTERNAL plane (0 < u < 1) translated
 * by +eps/-eps along its unit normal (the direction of increasing u).  The both-test
 * is not widened.  A pair is grazing iff the hit flag differs between the two runs;
 * its value (t, u, n, kind) is ill-conditioned at the eps scale iff the two runs
 * disagree beyond the parity tolerance.  Both runs are returned.
 *
 * Precision: double throughout.  Inputs are the FP32 arrays promoted exactly.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_KIND_LATERAL 0
#define OR_KIND_CAP0 1
#define OR_KIND_CAP1 2
#define OR_KIND_WEDGE 3
#define OR_KIND_INSIDE 4

/* which constraint produced an interval bound */
#define TAG_ORIGIN 0   /* t >= 0 (ray origin)                      */
#define TAG_START 1    /* the fiber's global start plane (u = 0)   */
#define TAG_END 2      /* the fiber's global end plane   (u = 1)   */
#define TAG_INTERNAL 3 /* any plane at 0 < u < 1                   */
#define TAG_TMAX 4     /* t <= ray t_max                           */

/* ------------------------------------------------------------------ */
/* small vector helpers (double, 3 and 4 components)                   */
/* ------------------------------------------------------------------ */
static double dot3(const double a[3], const double b[3]) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}
static void cross3(const double a[3], const double b[3], double out[3]) {
  out[0] = a[1] * b[2] - a[2] * b[1];
  out[1] = a[2] * b[0] - a[0] * b[2];
  out[2] = a[0] * b[1] - a[1] * b[0];
}
static void sub3(const double a[3], const double b[3], double out[3]) {
  out[0] = a[0] - b[0];
  out[1] = a[1] - b[1];
  out[2] = a[2] - b[2];
}
static double norm3(const double a[3]) { return sqrt(dot3(a, a)); }

/* ------------------------------------------------------------------ */
/* curve evaluation -- lst:eval_cubic_bezier P:1347-1364               */
/* P is 4 control points x 4 components (x, y, z, radius)              */
/* ------------------------------------------------------------------ */
void oracle_eval(const double P[16], double u, double out[4]) {
  double v = 1.0 - u;
  double b0 = v * v * v, b1 = 3.0 * u * v * v, b2 = 3.0 * u * u * v, b3 = u * u * u;
  for (int k = 0; k < 4; ++k)
    out[k] = b0 * P[0 + k] + b1 * P[4 + k] + b2 * P[8 + k] + b3 * P[12 + k];
}

/* the listing's "(scaled) derivative": C'(u) / 3 -- P:1357-1363 */
void oracle_eval_derivative(const double P[16], double u, double out[4]) {
  double v = 1.0 - u;
  for (int k = 0; k < 4; ++k)
    out[k] = v * v * (P[4 + k] - P[0 + k]) + 2.0 * u * v * (P[8 + k] - P[4 + k]) +
             u * u * (P[12 + k] - P[8 + k]);
}

/* Control points of the sub-curve on [u0, u1] (lst:recalculation P:1371-1385):
 *   Q0 = C(u0), Q3 = C(u1), Q1 = Q0 + (u1-u0) C'(u0)/3, Q2 = Q3 - (u1-u0) C'(u1)/3. */
void oracle_subcurve(const double P[16], double u0, double u1, double Q[16]) {
  double h = u1 - u0, e0[4], e1[4], d0[4], d1[4];
  oracle_eval(P, u0, e0);
  oracle_eval(P, u1, e1);
  oracle_eval_derivative(P, u0, d0);
  oracle_eval_derivative(P, u1, d1);
  for (int k = 0; k < 4; ++k) {
    Q[0 + k] = e0[k];
    Q[4 + k] = e0[k] + h * d0[k];
    Q[8 + k] = e1[k] - h * d1[k];
    Q[12 + k] = e1[k];
  }
}

/* Distance of point x to the line through q along a (|a| > 0), else |x - q|. */
static double dist_point_line(const double x[3], const double q[3], const double a[3]) {
  double m[3], c[3];
  sub3(x, q, m);
  double la = norm3(a);
  if (la == 0.0) return norm3(m);
  cross3(m, a, c);
  return norm3(c) / la;
}

/* Conservative radius of the bounding cylinder of sub-curve Q (P:488-495,
 * lst:calc_radius P:1415-1425): largest distance of the inner control points to
 * the chord Q0->Q3 plus the largest radius control point. */
double oracle_conservative_radius(const double Q[16]) {
  double a[3];
  sub3(&Q[12], &Q[0], a);
  double d1 = dist_point_line(&Q[4], &Q[0], a);
  double d2 = dist_point_line(&Q[8], &Q[0], a);
  double rmax = fmax(fmax(Q[3], Q[7]), fmax(Q[11], Q[15]));
  return fmax(d1, d2) + rmax;
}

/* Parameter interval {t : dist(o + t w, line(q, a)) <= R} of an infinite
 * cylinder.  Written in the closest-approach form of Appendix A: with
 * n = w x a^, the squared line-line distance d^2 = <o - q, n>^2 / |n|^2 (eq. P:814), the
 * parameter of closest approach t_cpa and the half chord
 * s = sqrt((R^2 - d^2) / |n|^2), since |(o + t w - q) x a^|^2 =
 * d^2 + |n|^2 (t - t_cpa)^2.  (This form keeps full precision for rays that pass close to
 * tangency, where expanding the quadratic cancels.)  Returns 0 if empty, 1 if [*c0, *c1]
 * (c0 = -inf, c1 = +inf when the ray is parallel to the axis and inside, F4). */
int oracle_cylinder(const double o[3], const double w[3], const double q[3], const double a[3],
                    double R, double *c0, double *c1) {
  double la = norm3(a);
  double ah[3] = {a[0] / la, a[1] / la, a[2] / la};
  double m[3], n[3], mx[3];
  sub3(o, q, m);
  cross3(w, ah, n); /* w x a^ */
  double A = dot3(n, n);
  if (A == 0.0) { /* F4: ray parallel to the axis */
    cross3(m, ah, mx);
    if (dot3(mx, mx) <= R * R) {
      *c0 = -INFINITY;
      *c1 = INFINITY;
      return 1;
    }
    return 0;
  }
  double mn = dot3(m, n);
  double d2 = mn * mn / A; /* squared distance between the ray line and the axis */
  if (d2 > R * R) return 0;
  cross3(m, ah, mx);
  double tcpa = -dot3(mx, n) / A;
  double s = sqrt((R * R - d2) / A);
  *c0 = tcpa - s;
  *c1 = tcpa + s;
  return 1;
}

/* ------------------------------------------------------------------ */
/* intervals along the ray                                              */
/* ------------------------------------------------------------------ */
typedef struct {
  double lo, hi;
  int lo_tag, hi_tag;
  int empty; /* F3/F5: explicit emptiness */
} ival;

/* Intersect I with the half-space {t : alpha + beta t >= 0} (F3 for beta == 0). */
static void clip_halfspace(ival *I, double alpha, double beta, int tag) {
  if (beta > 0.0) {
    double t = -alpha / beta;
    if (t > I->lo) {
      I->lo = t;
      I->lo_tag = tag;
    }
  } else if (beta < 0.0) {
    double t = -alpha / beta;
    if (t < I->hi) {
      I->hi = t;
      I->hi_tag = tag;
    }
  } else if (alpha < 0.0) {
    I->empty = 1;
  }
}

/* ------------------------------------------------------------------ */
/* the recursion                                                        */
/* ------------------------------------------------------------------ */
typedef struct {
  double P[16]; /* control points (x, y, z, r) x 4 */
  double o[3], w[3], tmax;
  int D;
  double eps;   /* grazing perturbation distance            */
  int eps_sign; /* 0 exact, +1 grow volumes, -1 shrink them */
  /* counters */
  int tests, descents, backtracks;
  /* optional trace of visited nodes: (level, u0, u1, event) */
  int trace_cap, trace_n;
  double *trace;
} octx;

typedef struct {
  int hit;
  double t;
  int kind;
  double u0, u1; /* leaf */
  double lo;
} ores;

static void trace_push(octx *c, int level, double u0, double u1, int ev) {
  if (c->trace && c->trace_n < c->trace_cap) {
    double *r = c->trace + 4 * c->trace_n;
    r[0] = level;
    r[1] = u0;
    r[2] = u1;
    r[3] = ev;
    c->trace_n++;
  }
}

/* Slab(N) = [0, t_max] cut by the node's start and end planes (lst:calc_t_interval
 * P:1459-1477; F7).  Start plane through Q0 with normal Q1-Q0 keeps <x-Q0,n0> >= 0;
 * end plane through Q3 with normal Q3-Q2 keeps <x-Q3,n1> <= 0. */
static ival slab(const octx *c, const double Q[16], double u0, double u1) {
  ival I = {0.0, c->tmax, TAG_ORIGIN, TAG_TMAX, 0};
  double n0[3], n1[3], m[3];
  sub3(&Q[4], &Q[0], n0);
  sub3(&Q[12], &Q[8], n1);
  double sh = c->eps_sign * c->eps;
  /* global cap: grow (+) / shrink (-); internal plane: translate along +n by sh */
  sub3(c->o, &Q[0], m);
  clip_halfspace(&I, dot3(m, n0) + (u0 == 0.0 ? sh : -sh) * norm3(n0), dot3(c->w, n0),
                 u0 == 0.0 ? TAG_START : TAG_INTERNAL);
  sub3(c->o, &Q[12], m);
  clip_halfspace(&I, -dot3(m, n1) + sh * norm3(n1), -dot3(c->w, n1),
                 u1 == 1.0 ? TAG_END : TAG_INTERNAL);
  return I;
}

static ores visit(octx *c, int level, double u0, double u1, ival I) {
  ores miss = {0, 0.0, 0, u0, u1, 0.0};
  double Q[16], a[3], c0, c1;
  c->tests++;
  oracle_subcurve(c->P, u0, u1, Q);
  sub3(&Q[12], &Q[0], a);
  double R = oracle_conservative_radius(Q) + c->eps_sign * c->eps;
  int nonempty = (R >= 0.0) && oracle_cylinder(c->o, c->w, &Q[0], a, R, &c0, &c1);
  /* 1. pruning test with F1 and F5 */
  if (!nonempty || I.empty || c1 < I.lo || c0 > I.hi || I.lo > I.hi) {
    trace_push(c, level, u0, u1, 0);
    return miss;
  }
  /* 2. leaf: first hit terminates, entry into the cropped cylinder (F2) */
  if (level == c->D) {
    trace_push(c, level, u0, u1, 2);
    ores r;
    r.hit = 1;
    r.u0 = u0;
    r.u1 = u1;
    r.lo = I.lo;
    if (c0 >= I.lo) {
      r.t = c0;
      r.kind = OR_KIND_LATERAL;
    } else {
      r.t = I.lo;
      if (I.lo_tag == TAG_ORIGIN)
        r.kind = OR_KIND_INSIDE;
      else if (I.lo_tag == TAG_START && u0 == 0.0)
        r.kind = OR_KIND_CAP0;
      else if (I.lo_tag == TAG_END && u1 == 1.0)
        r.kind = OR_KIND_CAP1;
      else
        r.kind = OR_KIND_WEDGE;
    }
    return r;
  }
  c->descents++;
  /* 3. partition plane through the split point S = C(um), normal n = C'(um)
   *    (3.2 P:455-456, 3.1 P:376-379).  sigma(t) = <o + t w - S, n>. */
  double um = 0.5 * (u0 + u1), S[4], n[4], m[3];
  oracle_eval(c->P, um, S);
  oracle_eval_derivative(c->P, um, n);
  sub3(c->o, S, m);
  /* eps runs: the internal plane is translated by eps_sign * eps along n^ */
  double alpha = dot3(m, n) - c->eps_sign * c->eps * norm3(n), beta = dot3(c->w, n);
  int right, both;
  ival In = I;
  if (beta != 0.0) {
    double tP = -alpha / beta;
    double sig; /* sign of sigma at the cylinder entry c0 */
    if (isinf(c0))
      sig = -beta; /* sigma(-inf) has the sign of -beta */
    else
      sig = alpha + beta * c0;
    /* near child first (F9); tie -> the child the ray continues into */
    right = (sig > 0.0) || (sig == 0.0 && beta > 0.0);
    /* both children only if the plane is crossed inside the UNCROPPED cylinder
     * */
    both = (c0 < tP) && (tP < c1);
    /* one-bound update */
    if (tP > c0) {
      if (tP < In.hi) {
        In.hi = tP;
        In.hi_tag = TAG_INTERNAL;
      }
    } else {
      if (tP > In.lo) {
        In.lo = tP;
        In.lo_tag = TAG_INTERNAL;
      }
    }
  } else {
    /* F3: plane parallel to the ray -- the ray lies wholly on one side */
    right = alpha > 0.0;
    both = 0;
  }
  /* event 1: descend, far child pruned; 3: descend, far child pending (both) */
  trace_push(c, level, u0, u1, both ? 3 : 1);
  double nu0 = right ? um : u0, nu1 = right ? u1 : um;
  ores r = visit(c, level + 1, nu0, nu1, In);
  if (r.hit) return r;
  if (!both) return miss;
  /* 7. far child with its own slab (F7) */
  c->backtracks++;
  double fu0 = right ? u0 : um, fu1 = right ? um : u1, Qf[16];
  oracle_subcurve(c->P, fu0, fu1, Qf);
  return visit(c, level + 1, fu0, fu1, slab(c, Qf, fu0, fu1));
}

/* Result of one pair: t, u, normal (lst:calc_intersection P:1546-1587 with F6, F8). */
typedef struct {
  double t, u, n[3];
  int hit, kind, tests, backtracks;
  double leaf_u0, leaf_u1;
} opair;

static opair run_pair(octx *c) {
  opair out;
  memset(&out, 0, sizeof(out));
  c->tests = c->descents = c->backtracks = 0;
  double Q[16];
  oracle_subcurve(c->P, 0.0, 1.0, Q);
  ores r = visit(c, 0, 0.0, 1.0, slab(c, Q, 0.0, 1.0));
  out.tests = c->tests;
  out.backtracks = c->backtracks;
  out.t = INFINITY;
  /* hit only strictly before t_max (F5) */
  if (!r.hit || !(r.t < c->tmax)) return out;
  out.hit = 1;
  out.t = r.t;
  out.kind = r.kind;
  out.leaf_u0 = r.u0;
  out.leaf_u1 = r.u1;
  double X[3] = {c->o[0] + r.t * c->w[0], c->o[1] + r.t * c->w[1], c->o[2] + r.t * c->w[2]};
  double L[16], a[3], xm[3];
  oracle_subcurve(c->P, r.u0, r.u1, L);
  sub3(&L[12], &L[0], a);
  sub3(X, &L[0], xm);
  double aa = dot3(a, a);
  double ul = aa > 0.0 ? dot3(xm, a) / aa : 0.0;
  ul = fmax(0.0, fmin(1.0, ul));
  if (r.kind == OR_KIND_CAP0) {
    out.u = 0.0;
    sub3(&c->P[0], &c->P[4], out.n);
  } else if (r.kind == OR_KIND_CAP1) {
    out.u = 1.0;
    sub3(&c->P[12], &c->P[8], out.n);
  } else {
    out.u = r.u0 + ul * (r.u1 - r.u0);
    for (int k = 0; k < 3; ++k) out.n[k] = X[k] - (L[k] + ul * a[k]);
  }
  double nn = norm3(out.n);
  if (nn > 0.0)
    for (int k = 0; k < 3; ++k) out.n[k] /= nn;
  return out;
}

/* ------------------------------------------------------------------ */
/* grazing band width (R5)                          */
/* eps = max(eps_rel_r * r_max, eps_ulps * 2^-52 * S_pair): the north star's 1e-6 r band,
 * with an FP64-rounding floor; S_pair = largest |coordinate|
 * of the control points relative to o' = o + <c - o, w^> w^, c = (P0+P3)/2 */
/* ------------------------------------------------------------------ */
static double pair_eps(const octx *c, double eps_rel_r, double eps_ulps) {
  double lw = norm3(c->w);
  double wh[3] = {c->w[0] / lw, c->w[1] / lw, c->w[2] / lw};
  double cm[3], m[3];
  for (int k = 0; k < 3; ++k) cm[k] = 0.5 * (c->P[k] + c->P[12 + k]);
  sub3(cm, c->o, m);
  double ts = dot3(m, wh);
  double op[3] = {c->o[0] + ts * wh[0], c->o[1] + ts * wh[1], c->o[2] + ts * wh[2]};
  double S = 0.0, rmax = 0.0;
  for (int i = 0; i < 4; ++i) {
    for (int k = 0; k < 3; ++k) S = fmax(S, fabs(c->P[4 * i + k] - op[k]));
    rmax = fmax(rmax, c->P[4 * i + 3]);
  }
  return fmax(eps_rel_r * rmax, eps_ulps * ldexp(1.0, -52) * S);
}

/* ------------------------------------------------------------------ */
/* public entry points (ctypes)                                         */
/* ------------------------------------------------------------------ */

/* Output record, one per pair (all doubles for simplicity):
 *  [0] t (inf on miss)  [1] u  [2..4] normal  [5] hit  [6] kind
 *  [7] node tests  [8] backtracks  [9] leaf u0  [10] leaf u1
 *  [11] grazing (hit(+eps) != hit(-eps))  [12] kind unstable (kind(+eps) != kind(-eps))
 *  [13] eps used
 *  [14..19] the +eps run: t, u, n[3], kind    [20..25] the -eps run: t, u, n[3], kind */
#define OREC 26

typedef struct {
  const float *rays;
  const float *ctrl, *radii;
  const uint32_t *pairs;
  int64_t n_rays, n_segs, n_pairs;
  int D, with_eps, degree;
  double eps_rel_r, eps_ulps;
  double *out;
  int64_t begin, end;
} job;

/* Degree elevation of a quadratic (q0, q1, q2) to the cubic (q0, (q0 + 2 q1)/3,
 * (2 q1 + q2)/3, q2) -- the same curve (and radius function), so the cubic method applies
 * unchanged (quadratic fibers, P:707 and App. B.1).  In FP64
 * from the FP32 inputs.  q: 3 points of 4 doubles (x, y, z, r); P: 4 points of 4. */
static void elevate_quadratic(const double q[12], double P[16]) {
  for (int k = 0; k < 4; ++k) {
    P[k] = q[k];
    P[4 + k] = (q[k] + 2.0 * q[4 + k]) / 3.0;
    P[8 + k] = (2.0 * q[4 + k] + q[8 + k]) / 3.0;
    P[12 + k] = q[8 + k];
  }
}

static void load_ctx(octx *c, const job *j, int64_t i) {
  uint32_t ri = j->pairs[2 * i], si = j->pairs[2 * i + 1];
  const float *ry = j->rays + 8 * (int64_t)ri;
  for (int k = 0; k < 3; ++k) {
    c->o[k] = ry[k];
    c->w[k] = ry[4 + k];
  }
  c->tmax = ry[3];
  if (j->degree == 2) {
    const float *cp = j->ctrl + 9 * (int64_t)si;
    const float *rr = j->radii + 3 * (int64_t)si;
    double q[12];
    for (int p = 0; p < 3; ++p) {
      for (int k = 0; k < 3; ++k) q[4 * p + k] = cp[3 * p + k];
      q[4 * p + 3] = rr[p];
    }
    elevate_quadratic(q, c->P);
  } else {
    const float *cp = j->ctrl + 12 * (int64_t)si;
    const float *rr = j->radii + 4 * (int64_t)si;
    for (int p = 0; p < 4; ++p) {
      for (int k = 0; k < 3; ++k) c->P[4 * p + k] = cp[3 * p + k];
      c->P[4 * p + 3] = rr[p];
    }
  }
  c->D = j->D;
  c->eps = 0.0;
  c->eps_sign = 0;
  c->trace = NULL;
  c->trace_cap = c->trace_n = 0;
}

static void *worker(void *arg) {
  const job *j = (const job *)arg;
  for (int64_t i = j->begin; i < j->end; ++i) {
    double *o = j->out + OREC * i;
    uint32_t ri = j->pairs[2 * i], si = j->pairs[2 * i + 1];
    memset(o, 0, sizeof(double) * OREC);
    if ((int64_t)ri >= j->n_rays || (int64_t)si >= j->n_segs) {
      o[0] = INFINITY;
      continue;
    }
    octx c;
    load_ctx(&c, j, i);
    opair r = run_pair(&c);
    o[0] = r.t;
    o[1] = r.u;
    o[2] = r.n[0];
    o[3] = r.n[1];
    o[4] = r.n[2];
    o[5] = r.hit;
    o[6] = r.kind;
    o[7] = r.tests;
    o[8] = r.backtracks;
    o[9] = r.leaf_u0;
    o[10] = r.leaf_u1;
    o[11] = 0;
    o[12] = 0;
    o[13] = 0;
    if (j->with_eps) {
      double eps = pair_eps(&c, j->eps_rel_r, j->eps_ulps);
      c.eps = eps;
      c.eps_sign = +1;
      opair rp = run_pair(&c);
      c.eps_sign = -1;
      opair rm = run_pair(&c);
      o[11] = (rp.hit != rm.hit);
      o[12] = (rp.hit && rm.hit && rp.kind != rm.kind) || (rp.hit != rm.hit);
      o[13] = eps;
      const opair *pm[2] = {&rp, &rm};
      for (int q = 0; q < 2; ++q) {
        double *e = o + 14 + 6 * q;
        e[0] = pm[q]->t;
        e[1] = pm[q]->u;
        e[2] = pm[q]->n[0];
        e[3] = pm[q]->n[1];
        e[4] = pm[q]->n[2];
        e[5] = pm[q]->hit ? pm[q]->kind : -1;
      }
    }
  }
  return NULL;
}

/* rays: f32[n_rays][8] = (ox, oy, oz, tmax, dx, dy, dz, pad); ctrl: f32[n_segs][4][3];
 * radii: f32[n_segs][4]; pairs: u32[n_pairs][2] = (ray, seg); out: f64[n_pairs][OREC].
 * with_eps: also run the +eps / -eps classification.  Returns 0, or -1 on bad args. */
int oracle_intersect_deg(const float *rays, int64_t n_rays, const float *ctrl,
                         const float *radii, int64_t n_segs, int degree, const uint32_t *pairs,
                         int64_t n_pairs, int depth, int with_eps, double eps_rel_r,
                         double eps_ulps, int nthreads, double *out) {
  if (depth < 0 || depth > 23 || n_pairs < 0 || (degree != 2 && degree != 3) ||
      (n_pairs > 0 && (!rays || !ctrl || !radii || !pairs || !out)))
    return -1;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if ((int64_t)nthreads > n_pairs) nthreads = n_pairs > 0 ? (int)n_pairs : 1;
  job jobs[256];
  pthread_t th[256];
  int64_t chunk = (n_pairs + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    job *j = &jobs[t];
    j->rays = rays;
    j->ctrl = ctrl;
    j->radii = radii;
    j->pairs = pairs;
    j->n_rays = n_rays;
    j->n_segs = n_segs;
    j->n_pairs = n_pairs;
    j->D = depth;
    j->with_eps = with_eps;
    j->degree = degree;
    j->eps_rel_r = eps_rel_r;
    j->eps_ulps = eps_ulps;
    j->out = out;
    j->begin = t * chunk;
    j->end = (t + 1) * chunk < n_pairs ? (t + 1) * chunk : n_pairs;
    if (j->begin > j->end) j->begin = j->end;
  }
  if (nthreads == 1) {
    worker(&jobs[0]);
    return 0;
  }
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, worker, &jobs[t]);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  return 0;
}

/* Cubic segments: ctrl f32[n_segs][4][3], radii f32[n_segs][4]. */
int oracle_intersect(const float *rays, int64_t n_rays, const float *ctrl, const float *radii,
                     int64_t n_segs, const uint32_t *pairs, int64_t n_pairs, int depth,
                     int with_eps, double eps_rel_r, double eps_ulps, int nthreads, double *out) {
  return oracle_intersect_deg(rays, n_rays, ctrl, radii, n_segs, 3, pairs, n_pairs, depth,
                              with_eps, eps_rel_r, eps_ulps, nthreads, out);
}

/* Single pair with an event trace: trace f64[cap][4] rows (level, u0, u1, event)
 * with event 0 = pruned, 1 = descended (far pruned), 3 = descended (far pending),
 * 2 = leaf hit.  out f64[OREC]
 * (no eps fields).  Returns the number of trace rows written. */
int oracle_trace(const float ray[8], const float ctrl[12], const float radii[4], int depth,
                 double eps_sign_eps, double *trace, int cap, double *out) {
  octx c;
  for (int k = 0; k < 3; ++k) {
    c.o[k] = ray[k];
    c.w[k] = ray[4 + k];
  }
  c.tmax = ray[3];
  for (int p = 0; p < 4; ++p) {
    for (int k = 0; k < 3; ++k) c.P[4 * p + k] = ctrl[3 * p + k];
    c.P[4 * p + 3] = radii[p];
  }
  c.D = depth;
  c.eps = fabs(eps_sign_eps);
  c.eps_sign = eps_sign_eps > 0 ? 1 : (eps_sign_eps < 0 ? -1 : 0);
  c.trace = trace;
  c.trace_cap = cap;
  c.trace_n = 0;
  opair r = run_pair(&c);
  out[0] = r.t;
  out[1] = r.u;
  out[2] = r.n[0];
  out[3] = r.n[1];
  out[4] = r.n[2];
  out[5] = r.hit;
  out[6] = r.kind;
  out[7] = r.tests;
  out[8] = r.backtracks;
  out[9] = r.leaf_u0;
  out[10] = r.leaf_u1;
  return c.trace_n;
}

/* The five cubic constraints of 3.4 (App. B eqs) on the
 * positions of P (f64[4][3]).  Returns a bitmask of VIOLATED inequalities
 * (bit k = inequality k+1 in the paper's order). */
int oracle_constraints(const double P[12]) {
  const double *p0 = P, *p1 = P + 3, *p2 = P + 6, *p3 = P + 9;
  double a[3], b[3];
  int bad = 0;
  sub3(p2, p0, a); sub3(p1, p0, b); if (dot3(a, b) < 0) bad |= 1;  /* <p2-p0, p1-p0> >= 0 */
  sub3(p3, p1, a); sub3(p1, p0, b); if (dot3(a, b) < 0) bad |= 2;  /* <p3-p1, p1-p0> >= 0 */
  sub3(p3, p1, a); sub3(p3, p2, b); if (dot3(a, b) < 0) bad |= 4;  /* <p3-p1, p3-p2> >= 0 */
  sub3(p2, p0, a); sub3(p3, p2, b); if (dot3(a, b) < 0) bad |= 8;  /* <p2-p0, p3-p2> >= 0 */
  sub3(p2, p0, a); sub3(p3, p1, b); if (dot3(a, b) < 0) bad |= 16; /* <p2-p0, p3-p1> >= 0 */
  return bad;
}

/* ------------------------------------------------------------------ */
/* input gatekeeper: thick-fiber / cusp test and    */
/* pre-splitting (3.4 P:609-703)                                        */
/* ------------------------------------------------------------------ */

/* rho(u) for the end plane through p_e with outward unit normal te: the
 * normal disc at u (centre C(u), normal C'(u)) reaches across the plane exactly when its
 * radius exceeds
 *   rho(u) = -<C(u) - p_e, te> / <n^_u, te>,   <n^_u, te> = |C'(u) x te| / |C'(u)|,
 * n_u = te - <te, t^_u> t^_u being the Gram-Schmidt displacement of P:676-682 (the disc's
 * point furthest along te is C(u) + r n^_u).  +inf where the disc is parallel to the plane
 * and the centre is inside; -inf where the centre itself is across. */
static double end_rho(const double P[16], double u, const double pe[3], const double te[3]) {
  double c[4], d[4], x[3], m[3];
  oracle_eval(P, u, c);
  oracle_eval_derivative(P, u, d);
  sub3(c, pe, m);
  cross3(d, te, x);
  double along = dot3(m, te);
  double s = norm3(x) / norm3(d);
  if (s == 0.0) return along <= 0.0 ? INFINITY : -INFINITY;
  return -along / s;
}

/* Thick-fiber / cusp margin of one end ("check each fiber only initially in its
 * two end points"): s* = inf over u in [0, 1) of rho(u) / r(u), with r(u) = the
 * largest radius control point r_bar ("or just ... r_u <= r_bar") or, parametric = 1,
 * the cubic radius itself.  The surface crosses the end plane (a valid part would be
 * cropped) iff s* < 1.  end = 1: the plane through p3 with normal p3 - p2;
 * end = 0: the plane through p0 with normal p0 - p1 (the reversed curve).
 * Computed plainly: 4096 uniform samples, 26 samples approaching the end (1 - 2^-j) and the
 * end limit rho(1) = 1 / curvature(1) = |C'|^3 / |C' x C''| (both numerator and
 * denominator of rho vanish there), then golden-section refinement around the smallest
 * sample.  Returns +inf for a straight segment. */
static double margin_ratio(const double P[16], double u, int parametric, double rbar,
                           double rho) {
  double r = rbar;
  if (parametric) {
    double c[4];
    oracle_eval(P, u, c);
    r = c[3];
  }
  return r > 0.0 ? rho / r : INFINITY;
}

double oracle_end_margin(const double P_in[16], int end, int parametric) {
  double P[16];
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < 4; ++k) P[4 * i + k] = end ? P_in[4 * i + k] : P_in[4 * (3 - i) + k];
  const double *pe = &P[12];
  double te[3];
  sub3(&P[12], &P[8], te);
  double lt = norm3(te);
  if (lt == 0.0) return -INFINITY;  /* degenerate end tangent: no plane */
  for (int k = 0; k < 3; ++k) te[k] /= lt;
  double rbar = fmax(fmax(P[3], P[7]), fmax(P[11], P[15]));
  double best = INFINITY, bu = 0.0;
  const int N = 4096;
  for (int i = 0; i < N; ++i) {
    double u = (double)i / N;
    double v = margin_ratio(P, u, parametric, rbar, end_rho(P, u, pe, te));
    if (v < best) best = v, bu = u;
  }
  for (int j = 1; j <= 26; ++j) {
    double u = 1.0 - ldexp(1.0, -j);
    double v = margin_ratio(P, u, parametric, rbar, end_rho(P, u, pe, te));
    if (v < best) best = v, bu = u;
  }
  /* the end limit: C'(1) = 3 (p3 - p2), C''(1) = 6 (p3 - 2 p2 + p1) */
  {
    double d1[3], d2[3], x[3];
    for (int k = 0; k < 3; ++k) {
      d1[k] = 3.0 * (P[12 + k] - P[8 + k]);
      d2[k] = 6.0 * (P[12 + k] - 2.0 * P[8 + k] + P[4 + k]);
    }
    cross3(d1, d2, x);
    double l1 = norm3(d1), lx = norm3(x);
    double rho1 = lx > 0.0 ? l1 * l1 * l1 / lx : INFINITY;
    double v = margin_ratio(P, 1.0, parametric, rbar, rho1);
    if (v < best) best = v, bu = 1.0;
  }
  if (bu < 1.0 && isfinite(best)) {
    /* golden-section refinement of the ratio on the bracket around the best sample */
    double a = fmax(0.0, bu - 1.0 / N), b = fmin(1.0 - ldexp(1.0, -30), bu + 1.0 / N);
    const double g = 0.5 * (sqrt(5.0) - 1.0);
    double x1 = b - g * (b - a), x2 = a + g * (b - a);
    double f1 = margin_ratio(P, x1, parametric, rbar, end_rho(P, x1, pe, te));
    double f2 = margin_ratio(P, x2, parametric, rbar, end_rho(P, x2, pe, te));
    for (int it = 0; it < 100; ++it) {
      if (f1 < f2) {
        b = x2, x2 = x1, f2 = f1, x1 = b - g * (b - a);
        f1 = margin_ratio(P, x1, parametric, rbar, end_rho(P, x1, pe, te));
      } else {
        a = x1, x1 = x2, f1 = f2, x2 = a + g * (b - a);
        f2 = margin_ratio(P, x2, parametric, rbar, end_rho(P, x2, pe, te));
      }
    }
    best = fmin(best, fmin(f1, f2));
  }
  return best;
}

/* One segment passes the gatekeeper (3.4 P:609-703): the five constraints hold and neither
 * end plane is crossed by the surface (margin >= 1 at both ends). */
static int piece_valid(const double Q[16], int parametric) {
  double pos[12];
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < 3; ++k) pos[3 * i + k] = Q[4 * i + k];
  if (oracle_constraints(pos)) return 0;
  return oracle_end_margin(Q, 0, parametric) >= 1.0 && oracle_end_margin(Q, 1, parametric) >= 1.0;
}

/* Pre-splitting ("must be subdivided beforehand"): bisect at
 * the parameter midpoint (de Casteljau, via oracle_subcurve) until every piece passes
 * piece_valid or max_level halvings are reached.  Writes the pieces in curve order as
 * (u0, u1, valid) triples into out[3 * k ...] (at most cap pieces) and returns their
 * number (or -1 if cap is too small).  The pieces tile [0, 1]. */
static int presplit_rec(const double P[16], double u0, double u1, int level, int max_level,
                        int parametric, double *out, int cap, int n) {
  if (n < 0) return n;
  double Q[16];
  oracle_subcurve(P, u0, u1, Q);
  int ok = piece_valid(Q, parametric);
  if (ok || level >= max_level) {
    if (n >= cap) return -1;
    out[3 * n] = u0;
    out[3 * n + 1] = u1;
    out[3 * n + 2] = ok;
    return n + 1;
  }
  double um = 0.5 * (u0 + u1);
  n = presplit_rec(P, u0, um, level + 1, max_level, parametric, out, cap, n);
  return presplit_rec(P, um, u1, level + 1, max_level, parametric, out, cap, n);
}

int oracle_presplit(const double P[16], int max_level, int parametric, double *out, int cap) {
  return presplit_rec(P, 0.0, 1.0, 0, max_level, parametric, out, cap, 0);
}

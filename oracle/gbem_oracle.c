/* gbem_oracle.c — TEST INFRASTRUCTURE ONLY: CPU restatement of the reference
 * single-layer Galerkin path (see gbem_oracle.h).  Never shipped; the product
 * path (paper_2203_11733_b200/) neither links nor loads this file.
 *
 * Every function names the reference lines it restates.  Arithmetic is written
 * in the reference's evaluation order so that, compiled without FP contraction
 * (oracle/Makefile passes -ffp-contract=off), results are bit-identical to the
 * reference headers compiled into oracle/_ref with the same flags.
 */
#include "gbem_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* kFourPi (oracle.hpp:11) */
static const double kFourPi = 4.0 * 3.14159265358979323846;

/* ---------------- geometry helpers (geometry.hpp:21-87) ---------------- */

typedef struct {
  double lo, hi;
} span_t;

static span_t rect_extent(const orc_rect* r, int k) {
  /* Rect::extent (geometry.hpp:62-66) with inplaneAxes (geometry.hpp:41-47) */
  span_t s;
  if (k == r->axis) {
    s.lo = r->level;
    s.hi = r->level;
    return s;
  }
  int first = (r->axis == 0) ? 1 : 0;
  if (k == first) {
    s.lo = r->a0;
    s.hi = r->a1;
  } else {
    s.lo = r->b0;
    s.hi = r->b1;
  }
  return s;
}

double orc_rect_distance(const orc_rect* a, const orc_rect* b) {
  /* rectDistance (geometry.hpp:79-87) */
  double s = 0.0;
  for (int k = 0; k < 3; ++k) {
    span_t ea = rect_extent(a, k), eb = rect_extent(b, k);
    double g = eb.lo - ea.hi;
    double g2 = ea.lo - eb.hi;
    if (g2 > g) g = g2;
    if (0.0 > g) g = 0.0;
    s += g * g;
  }
  return sqrt(s);
}

double orc_rect_diameter(const orc_rect* a) { return hypot(a->a1 - a->a0, a->b1 - a->b0); }

/* ---------------- quadrature (quadrature.hpp) ---------------- */

typedef double (*integrand_fn)(const void* ctx, double x);

typedef struct {
  long evals;
  int converged;
  int status; /* 2 = non-finite sample */
} qstats;

#define ROMB_MAX 40

/* romberg (quadrature.hpp:27-64): trapezoid + Richardson; converged once the
 * diagonal moves by <= relTol*|T_kk| twice in a row past level 4. */
static double romberg(integrand_fn f, const void* ctx, double a, double b, double rel_tol,
                      int max_levels, qstats* st) {
  if (a == b) return 0.0;
  int L = max_levels;
  double rowA[ROMB_MAX + 1], rowB[ROMB_MAX + 1];
  double* prev = rowA;
  double* cur = rowB;
  double fa = f(ctx, a), fb = f(ctx, b);
  st->evals += 2;
  if (!isfinite(fa) || !isfinite(fb)) {
    st->status = 2;
    return NAN;
  }
  double h = b - a;
  prev[0] = 0.5 * h * (fa + fb);
  int hits = 0;
  for (int k = 1; k <= L; ++k) {
    h *= 0.5;
    double tot = 0.0;
    long n = 1L << k;
    for (long i = 1; i < n; i += 2) {
      double s = f(ctx, a + (double)i * h);
      ++st->evals;
      if (!isfinite(s)) {
        st->status = 2;
        return NAN;
      }
      tot += s;
    }
    cur[0] = 0.5 * prev[0] + h * tot;
    double p4 = 1.0;
    for (int m = 1; m <= k; ++m) {
      p4 *= 4.0;
      cur[m] = cur[m - 1] + (cur[m - 1] - prev[m - 1]) / (p4 - 1.0);
    }
    if (k >= 4) {
      double diff = fabs(cur[k] - prev[k - 1]);
      double mag = fabs(cur[k]);
      if (mag < 1e-300) mag = 1e-300;
      hits = diff <= rel_tol * mag ? hits + 1 : 0;
      if (hits >= 2) return cur[k];
    }
    double* t = prev;
    prev = cur;
    cur = t;
  }
  st->converged = 0;
  return prev[L];
}

/* t^4 endpoint substitution wrapper (quadrature.hpp:80-93) */
typedef struct {
  integrand_fn f;
  const void* ctx;
  double base;
  int from_hi; /* 0: f(a + t^4), 1: f(b - t^4) */
} t4_ctx;

static double t4_eval(const void* vc, double t) {
  const t4_ctx* c = (const t4_ctx*)vc;
  if (t == 0.0) return 0.0;
  double t4 = t * t * t * t;
  double x = c->from_hi ? c->base - t4 : c->base + t4;
  return 4.0 * t * t * t * c->f(c->ctx, x);
}

/* integrateSegment (quadrature.hpp:70-94) */
static double integrate_segment(integrand_fn f, const void* ctx, double a, double b, int singA,
                                int singB, double rel_tol, int max_levels, qstats* st) {
  if (a == b) return 0.0;
  if (singA && singB) {
    double m = 0.5 * (a + b);
    double left = integrate_segment(f, ctx, a, m, 1, 0, rel_tol, max_levels, st);
    double right = integrate_segment(f, ctx, m, b, 0, 1, rel_tol, max_levels, st);
    return left + right;
  }
  if (singA || singB) {
    double L = b - a;
    t4_ctx c;
    c.f = f;
    c.ctx = ctx;
    c.base = singA ? a : b;
    c.from_hi = singA ? 0 : 1;
    return romberg(t4_eval, &c, 0.0, sqrt(sqrt(L)), rel_tol, max_levels, st);
  }
  return romberg(f, ctx, a, b, rel_tol, max_levels, st);
}

/* integrateWithSplits (quadrature.hpp:98-113): split at 0 when interior, probe
 * each endpoint for a non-finite value (probes are not counted as evals). */
static double integrate_with_splits(integrand_fn f, const void* ctx, double a, double b,
                                    double rel_tol, int max_levels, qstats* st) {
  double pts[3] = {a, b, 0.0};
  int n = 2;
  if (a < 0.0 && 0.0 < b) {
    pts[0] = a;
    pts[1] = 0.0;
    pts[2] = b;
    n = 3;
  }
  double total = 0.0;
  for (int i = 0; i + 1 < n; ++i) {
    int sa = !isfinite(f(ctx, pts[i]));
    int sb = !isfinite(f(ctx, pts[i + 1]));
    total += integrate_segment(f, ctx, pts[i], pts[i + 1], sa, sb, rel_tol, max_levels, st);
  }
  return total;
}

/* 6-node Gauss-Legendre (quadrature.hpp:116-124) */
static const double kGX[6] = {-0.9324695142031520278123016, -0.6612093864662645136613996,
                              -0.2386191860831969086305017, 0.2386191860831969086305017,
                              0.6612093864662645136613996,  0.9324695142031520278123016};
static const double kGW[6] = {0.1713244923791703450402961, 0.3607615730481386075698335,
                              0.4679139345726910473898703, 0.4679139345726910473898703,
                              0.3607615730481386075698335, 0.1713244923791703450402961};

/* ---------------- closed-form pieces (kernels.hpp:46-94) ---------------- */

/* logUPlusR (kernels.hpp:48-56): log(u + sqrt(u^2 + c2)), stable for u < 0 */
static double log_u_plus_r(double u, double c2) {
  double r = sqrt(u * u + c2);
  if (u >= 0.0) {
    double arg = u + r;
    return arg > 0.0 ? log(arg) : -INFINITY;
  }
  if (c2 == 0.0) return -INFINITY;
  return log(c2) - log(r - u);
}

/* mulLog (kernels.hpp:59-62) */
static double mul_log(double pref, double u, double c2, double guard) {
  if (fabs(pref) <= guard) return 0.0;
  return pref * log_u_plus_r(u, c2);
}

/* uCorners (kernels.hpp:71-73): signs (+,+,-,-) */
static void u_corners(double xd, double xu, double yd, double yu, double sign[4], double val[4]) {
  sign[0] = +1.0;
  val[0] = xu - yd;
  sign[1] = +1.0;
  val[1] = xd - yu;
  sign[2] = -1.0;
  val[2] = xu - yu;
  sign[3] = -1.0;
  val[3] = xd - yd;
}

/* kCoplanar (kernels.hpp:77-84) */
static double k_coplanar(double u, double v, double guard) {
  double s = sqrt(u * u + v * v);
  double g1 = mul_log(0.5 * u * v * v, u, v * v, guard) - 0.75 * u * v * v +
              mul_log(u * u * v, v, u * u, guard) - 0.5 * u * u * s;
  double g2 = (u * u + v * v) * s / 6.0 + mul_log(0.5 * u * u * v, v, u * u, guard) -
              0.5 * u * u * s;
  return g1 - g2;
}

static double max4(double a, double b, double c, double d) {
  /* std::max({a,b,c,d}) */
  double m = a;
  if (m < b) m = b;
  if (m < c) m = c;
  if (m < d) m = d;
  return m;
}

/* uCoplanar (kernels.hpp:86-94) */
static double u_coplanar(span_t sx, span_t sy, span_t tx, span_t ty) {
  double scale = max4(sx.hi - sx.lo, sy.hi - sy.lo, tx.hi - tx.lo, ty.hi - ty.lo);
  double guard = 1e-14 * scale * scale * scale;
  double su[4], vu[4], sv[4], vv[4];
  u_corners(sx.lo, sx.hi, tx.lo, tx.hi, su, vu);
  u_corners(sy.lo, sy.hi, ty.lo, ty.hi, sv, vv);
  double acc = 0.0;
  for (int p = 0; p < 4; ++p)
    for (int q = 0; q < 4; ++q) acc += su[p] * sv[q] * k_coplanar(vu[p], vv[q], guard);
  return acc / kFourPi;
}

/* ---------------- parallel offset (kernels.hpp:96-153) ---------------- */

typedef struct {
  double t0, t3, plateau;
} tent_t;

static double tent_w(const tent_t* w, double t) {
  /* Tent::operator() (kernels.hpp:101-103) */
  double m = t - w->t0;
  if (w->plateau < m) m = w->plateau;
  if (w->t3 - t < m) m = w->t3 - t;
  return m > 0.0 ? m : 0.0;
}

static int cmp_double(const void* x, const void* y) {
  double a = *(const double*)x, b = *(const double*)y;
  return (a > b) - (a < b);
}

/* tentSegments (kernels.hpp:112-125) */
static int tent_segments(double xd, double xu, double yd, double yu, tent_t* w, double cuts[5]) {
  double t0 = xd - yu, t3 = xu - yd;
  /* std::min(a,b) == (b < a ? b : a); std::max(a,b) == (a < b ? b : a) */
  double da = xd - yd, db = xu - yu;
  double k1 = db < da ? db : da;
  double k2 = da < db ? db : da;
  w->t0 = t0;
  w->t3 = t3;
  w->plateau = (yu - yd) < (xu - xd) ? (yu - yd) : (xu - xd);
  double pts[5] = {t0, k1, k2, t3, 0.0};
  int n = 4;
  if (t0 < 0.0 && 0.0 < t3) n = 5;
  qsort(pts, (size_t)n, sizeof(double), cmp_double);
  int count = 0;
  for (int i = 0; i < n; ++i)
    if (count == 0 || pts[i] > cuts[count - 1]) cuts[count++] = pts[i];
  return count;
}

typedef struct {
  double sign[4], val[4];
  double b2;
  tent_t w;
} par_ctx;

/* integrand of uParallelOffset (kernels.hpp:143-151) */
static double par_f(const void* vc, double v) {
  const par_ctx* c = (const par_ctx*)vc;
  double c2 = v * v + c->b2;
  double acc = 0.0;
  for (int k = 0; k < 4; ++k) {
    double u = c->val[k];
    double r = sqrt(u * u + c2);
    acc += c->sign[k] * (u * log_u_plus_r(u, c2) - r);
  }
  return tent_w(&c->w, v) * acc;
}

/* uParallelOffset (kernels.hpp:138-153) */
static double u_parallel_offset(span_t sx, span_t sy, span_t tx, span_t ty, double b,
                                double rel_tol, int max_levels, qstats* st) {
  par_ctx c;
  c.b2 = b * b;
  u_corners(sx.lo, sx.hi, tx.lo, tx.hi, c.sign, c.val);
  double cuts[5];
  int count = tent_segments(sy.lo, sy.hi, ty.lo, ty.hi, &c.w, cuts);
  double total = 0.0;
  for (int i = 0; i + 1 < count; ++i) {
    total += romberg(par_f, &c, cuts[i], cuts[i + 1], rel_tol, max_levels, st);
    if (st->status) return NAN;
  }
  return total / kFourPi;
}

/* ---------------- orthogonal (kernels.hpp:171-214, 239-255) ---------------- */

typedef struct {
  double sign[4], val[4];
  double x3d, x3u, y2d, y2u;
  double guard;
} orth_ctx;

/* fx of uOrthogonal (kernels.hpp:183-199) */
static double orth_fx(const void* vc, double x) {
  const orth_ctx* c = (const orth_ctx*)vc;
  double acc = 0.0;
  double x2 = x * x;
  for (int k = 0; k < 4; ++k) {
    double cv = c->val[k];
    double u2 = cv * cv;
    for (int side = 0; side < 2; ++side) {
      double sy = side == 0 ? +1.0 : -1.0;
      double y = side == 0 ? c->y2u : c->y2d;
      double c2 = x2 + y * y;
      double term = mul_log(0.5 * cv * y, cv, c2, c->guard) +
                    mul_log(0.5 * u2, y, u2 + x2, c->guard);
      double r = sqrt(u2 + c2);
      double g3 = 0.5 * y * r + mul_log(0.5 * (x2 + u2), y, u2 + x2, c->guard);
      acc += c->sign[k] * sy * (term - g3);
    }
  }
  return acc;
}

/* fy of uOrthogonal (kernels.hpp:201-210) */
static double orth_fy(const void* vc, double y) {
  const orth_ctx* c = (const orth_ctx*)vc;
  double acc = 0.0;
  double y2 = y * y;
  for (int k = 0; k < 4; ++k)
    for (int side = 0; side < 2; ++side) {
      double sx = side == 0 ? +1.0 : -1.0;
      double x = side == 0 ? c->x3u : c->x3d;
      double c2 = x * x + y2;
      acc += c->sign[k] * sx * mul_log(0.5 * c->val[k] * x, c->val[k], c2, c->guard);
    }
  return acc;
}

static double u_orthogonal(span_t s1, span_t s3, span_t t1, span_t t2, double rel_tol,
                           int max_levels, qstats* st) {
  orth_ctx c;
  u_corners(s1.lo, s1.hi, t1.lo, t1.hi, c.sign, c.val);
  c.x3d = s3.lo;
  c.x3u = s3.hi;
  c.y2d = t2.lo;
  c.y2u = t2.hi;
  double scale = max4(s1.hi - s1.lo, t1.hi - t1.lo, s3.hi - s3.lo, t2.hi - t2.lo);
  if (scale < 1e-30) scale = 1e-30;
  c.guard = 1e-14 * scale;
  double tx = integrate_with_splits(orth_fx, &c, c.x3d, c.x3u, rel_tol, max_levels, st);
  if (st->status) return NAN;
  double ty = integrate_with_splits(orth_fy, &c, t2.lo, t2.hi, rel_tol, max_levels, st);
  if (st->status) return NAN;
  return (tx + ty) / kFourPi;
}

/* rectLess (kernels.hpp:257-263): lexicographic (axis, level, a0, a1, b0, b1) */
static int rect_less(const orc_rect* a, const orc_rect* b) {
  double ka[6] = {(double)a->axis, a->level, a->a0, a->a1, a->b0, a->b1};
  double kb[6] = {(double)b->axis, b->level, b->a0, b->a1, b->b0, b->b1};
  for (int i = 0; i < 6; ++i) {
    if (ka[i] < kb[i]) return 1;
    if (kb[i] < ka[i]) return 0;
  }
  return 0;
}

orc_kv orc_u_pair_integral(const orc_rect* Ii, const orc_rect* Ij, double rel_tol,
                           int max_levels) {
  /* u_pair_integral (kernels.hpp:270-291): canonical argument order, then
   * coplanar / offset-parallel / orthogonal dispatch. */
  const orc_rect* a = rect_less(Ij, Ii) ? Ij : Ii;
  const orc_rect* b = rect_less(Ij, Ii) ? Ii : Ij;
  qstats st = {0, 1, 0};
  orc_kv out;
  if (max_levels > ROMB_MAX) max_levels = ROMB_MAX;
  span_t aA = {a->a0, a->a1}, aB = {a->b0, a->b1}, bA = {b->a0, b->a1}, bB = {b->b0, b->b1};
  if (a->axis == b->axis) {
    double off = a->level - b->level;
    if (off == 0.0)
      out.value = u_coplanar(aA, aB, bA, bB);
    else
      out.value = u_parallel_offset(aA, aB, bA, bB, off, rel_tol, max_levels, &st);
  } else {
    /* orthFrame (kernels.hpp:245-255) */
    int shared = 3 - a->axis - b->axis;
    span_t s1 = rect_extent(a, shared), t1 = rect_extent(b, shared);
    span_t i3 = rect_extent(a, b->axis), j2 = rect_extent(b, a->axis);
    span_t s3 = {i3.lo - b->level, i3.hi - b->level};
    span_t t2 = {j2.lo - a->level, j2.hi - a->level};
    out.value = u_orthogonal(s1, s3, t1, t2, rel_tol, max_levels, &st);
  }
  out.converged = st.converged;
  out.evals = st.evals;
  out.status = st.status;
  return out;
}

/* ---------------- double layer (kernels.hpp:157-169, 218-237, 295-315) ---------------- */

/* integrand of qParallelOffset (kernels.hpp:162-167) */
static double qpar_f(const void* vc, double v) {
  const par_ctx* c = (const par_ctx*)vc;
  double c2 = v * v + c->b2;
  double acc = 0.0;
  for (int k = 0; k < 4; ++k) acc += c->sign[k] * sqrt(c->val[k] * c->val[k] + c2) / c2;
  return tent_w(&c->w, v) * acc;
}

/* qParallelOffset (kernels.hpp:157-169): b = test level - source level */
static double q_parallel_offset(span_t sx, span_t sy, span_t tx, span_t ty, double b, double rel_tol,
                                int max_levels, qstats* st) {
  par_ctx c;
  c.b2 = b * b;
  u_corners(sx.lo, sx.hi, tx.lo, tx.hi, c.sign, c.val);
  double cuts[5];
  int count = tent_segments(sy.lo, sy.hi, ty.lo, ty.hi, &c.w, cuts);
  double total = 0.0;
  for (int i = 0; i + 1 < count; ++i) {
    total += romberg(qpar_f, &c, cuts[i], cuts[i + 1], rel_tol, max_levels, st);
    if (st->status) return NAN;
  }
  return b * total / kFourPi;
}

/* fy of qOrthogonal (kernels.hpp:224-235) */
static double qorth_fy(const void* vc, double y) {
  const orth_ctx* c = (const orth_ctx*)vc;
  double acc = 0.0;
  double y2 = y * y;
  for (int side = 0; side < 2; ++side) {
    double s3s = side == 0 ? +1.0 : -1.0;
    double x3 = side == 0 ? c->x3d : c->x3u;
    double c2 = y2 + x3 * x3;
    for (int k = 0; k < 4; ++k) {
      double r = sqrt(c->val[k] * c->val[k] + c2);
      acc += s3s * c->sign[k] * (mul_log(c->val[k], c->val[k], c2, c->guard) - r);
    }
  }
  return acc;
}

/* qOrthogonal (kernels.hpp:218-237) */
static double q_orthogonal(span_t s1, span_t s3, span_t t1, span_t t2, double rel_tol, int max_levels,
                           qstats* st) {
  orth_ctx c;
  u_corners(s1.lo, s1.hi, t1.lo, t1.hi, c.sign, c.val);
  c.x3d = s3.lo;
  c.x3u = s3.hi;
  c.y2d = t2.lo;
  c.y2u = t2.hi;
  double scale = max4(s1.hi - s1.lo, t1.hi - t1.lo, s3.hi - s3.lo, t2.hi - t2.lo);
  if (scale < 1e-30) scale = 1e-30;
  c.guard = 1e-14 * scale;
  double ty = integrate_with_splits(qorth_fy, &c, t2.lo, t2.hi, rel_tol, max_levels, st);
  if (st->status) return NAN;
  return ty / kFourPi;
}

orc_kv orc_q_pair_integral(const orc_rect* Ii, const orc_rect* Ij, int nsign_j, double rel_tol, int max_levels) {
  /* q_pair_integral (kernels.hpp:295-315): test Ii, source Ij with its normal
   * sign; no canonical reordering; coplanar pairs vanish. */
  qstats st = {0, 1, 0};
  orc_kv out;
  if (max_levels > ROMB_MAX) max_levels = ROMB_MAX;
  double ns = (double)nsign_j;
  span_t iA = {Ii->a0, Ii->a1}, iB = {Ii->b0, Ii->b1}, jA = {Ij->a0, Ij->a1}, jB = {Ij->b0, Ij->b1};
  if (Ii->axis == Ij->axis) {
    double off = Ii->level - Ij->level;
    out.value = off == 0.0 ? 0.0 : ns * q_parallel_offset(iA, iB, jA, jB, off, rel_tol, max_levels, &st);
  } else {
    int shared = 3 - Ii->axis - Ij->axis;
    span_t s1 = rect_extent(Ii, shared), t1 = rect_extent(Ij, shared);
    span_t i3 = rect_extent(Ii, Ij->axis), j2 = rect_extent(Ij, Ii->axis);
    span_t s3 = {i3.lo - Ij->level, i3.hi - Ij->level};
    span_t t2 = {j2.lo - Ii->level, j2.hi - Ii->level};
    out.value = ns * q_orthogonal(s1, s3, t1, t2, rel_tol, max_levels, &st);
  }
  out.converged = st.converged;
  out.evals = st.evals;
  out.status = st.status;
  return out;
}

/* ---------------- brute-force oracle (oracle.hpp:44-131,191-205) ---------------- */

static void gauss_nodes(double lo, double hi, double* x, double* w) {
  double c = 0.5 * (lo + hi), h = 0.5 * (hi - lo);
  for (int i = 0; i < 6; ++i) {
    x[i] = c + h * kGX[i];
    w[i] = h * kGW[i];
  }
}

/* gaussPair with UStar (oracle.hpp:45-88) */
static double gauss_pair6(const orc_rect* r1, const orc_rect* r2) {
  double xa[6], wa[6], xb[6], wb[6], xc[6], wc[6], xd[6], wd[6];
  gauss_nodes(r1->a0, r1->a1, xa, wa);
  gauss_nodes(r1->b0, r1->b1, xb, wb);
  gauss_nodes(r2->a0, r2->a1, xc, wc);
  gauss_nodes(r2->b0, r2->b1, xd, wd);
  int i1a = r1->axis == 0 ? 1 : 0, i1b = r1->axis == 2 ? 1 : 2;
  int i2a = r2->axis == 0 ? 1 : 0, i2b = r2->axis == 2 ? 1 : 2;
  double p[3] = {0, 0, 0}, q[3] = {0, 0, 0};
  p[r1->axis] = r1->level;
  q[r2->axis] = r2->level;
  double acc = 0.0;
  for (int i = 0; i < 6; ++i) {
    p[i1a] = xa[i];
    for (int j = 0; j < 6; ++j) {
      p[i1b] = xb[j];
      double w1 = wa[i] * wb[j];
      for (int k = 0; k < 6; ++k) {
        q[i2a] = xc[k];
        double w2 = w1 * wc[k];
        for (int l = 0; l < 6; ++l) {
          q[i2b] = xd[l];
          double dx = p[0] - q[0], dy = p[1] - q[1], dz = p[2] - q[2];
          acc += w2 * wd[l] * (1.0 / (kFourPi * sqrt(dx * dx + dy * dy + dz * dz)));
        }
      }
    }
  }
  return acc;
}

double orc_gauss_pair(const orc_rect* r1, const orc_rect* r2, int sub) {
  if (sub < 1) sub = 1;
  double acc = 0.0;
  double da1 = (r1->a1 - r1->a0) / sub, db1 = (r1->b1 - r1->b0) / sub;
  double da2 = (r2->a1 - r2->a0) / sub, db2 = (r2->b1 - r2->b0) / sub;
  for (int i = 0; i < sub; ++i)
    for (int j = 0; j < sub; ++j) {
      orc_rect c1 = *r1;
      c1.a0 = r1->a0 + da1 * i;
      c1.a1 = i + 1 == sub ? r1->a1 : r1->a0 + da1 * (i + 1);
      c1.b0 = r1->b0 + db1 * j;
      c1.b1 = j + 1 == sub ? r1->b1 : r1->b0 + db1 * (j + 1);
      for (int k = 0; k < sub; ++k)
        for (int l = 0; l < sub; ++l) {
          orc_rect c2 = *r2;
          c2.a0 = r2->a0 + da2 * k;
          c2.a1 = k + 1 == sub ? r2->a1 : r2->a0 + da2 * (k + 1);
          c2.b0 = r2->b0 + db2 * l;
          c2.b1 = l + 1 == sub ? r2->b1 : r2->b0 + db2 * (l + 1);
          acc += gauss_pair6(&c1, &c2);
        }
    }
  return acc;
}

static int same_geometry(const orc_rect* a, const orc_rect* b) {
  return a->axis == b->axis && a->level == b->level && a->a0 == b->a0 && a->a1 == b->a1 &&
         a->b0 == b->b0 && a->b1 == b->b1;
}

/* split4 (oracle.hpp:20-34) */
static void split4(const orc_rect* r, orc_rect out[4]) {
  double ma = 0.5 * (r->a0 + r->a1), mb = 0.5 * (r->b0 + r->b1);
  for (int k = 0; k < 4; ++k) out[k] = *r;
  out[0].a1 = ma;
  out[0].b1 = mb;
  out[1].a0 = ma;
  out[1].b1 = mb;
  out[2].a1 = ma;
  out[2].b0 = mb;
  out[3].a0 = ma;
  out[3].b0 = mb;
}

static orc_rect shifted(const orc_rect* r, double da, double db) {
  orc_rect s = *r;
  s.a0 = r->a0 + da;
  s.a1 = r->a1 + da;
  s.b0 = r->b0 + db;
  s.b1 = r->b1 + db;
  return s;
}

/* recU (oracle.hpp:105-131) */
static double rec_u(const orc_rect* r1, const orc_rect* r2, int depth) {
  if (same_geometry(r1, r2)) {
    orc_rect kids[4];
    split4(r1, kids);
    double w = 0.5 * (r1->a1 - r1->a0), h = 0.5 * (r1->b1 - r1->b0);
    orc_rect s1 = shifted(&kids[0], w, 0.0), s2 = shifted(&kids[0], 0.0, h),
             s3 = shifted(&kids[0], w, h);
    double a = rec_u(&kids[0], &s1, depth - 1);
    double b = rec_u(&kids[0], &s2, depth - 1);
    double c = rec_u(&kids[0], &s3, depth - 1);
    return 2.0 * (4.0 * a + 4.0 * b + 4.0 * c);
  }
  double d = orc_rect_distance(r1, r2);
  double d1 = orc_rect_diameter(r1), d2 = orc_rect_diameter(r2);
  double dm = d1 > d2 ? d1 : d2;
  if (d >= dm || depth <= 0) return gauss_pair6(r1, r2);
  if (d == 0.0) {
    orc_rect k1[4], k2[4];
    split4(r1, k1);
    split4(r2, k2);
    double acc = 0.0;
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) acc += rec_u(&k1[i], &k2[j], depth - 1);
    return acc;
  }
  double acc = 0.0;
  orc_rect k[4];
  if (d1 >= d2) {
    split4(r1, k);
    for (int i = 0; i < 4; ++i) acc += rec_u(&k[i], r2, depth - 1);
  } else {
    split4(r2, k);
    for (int i = 0; i < 4; ++i) acc += rec_u(r1, &k[i], depth - 1);
  }
  return acc;
}

/* cutSpan (oracle.hpp:134-144) */
static int cut_span(double lo, double hi, double c0, double c1, double out[4]) {
  double pts[4] = {lo, hi, 0, 0};
  int n = 2;
  if (c0 > lo && c0 < hi) pts[n++] = c0;
  if (c1 > lo && c1 < hi && c1 != c0) pts[n++] = c1;
  qsort(pts, (size_t)n, sizeof(double), cmp_double);
  for (int i = 0; i < n; ++i) out[i] = pts[i];
  return n - 1;
}

/* presplit (oracle.hpp:148-166) */
static int presplit(const orc_rect* r, const orc_rect* other, orc_rect out[9]) {
  int ia = r->axis == 0 ? 1 : 0, ib = r->axis == 2 ? 1 : 2;
  span_t oa = rect_extent(other, ia), ob = rect_extent(other, ib);
  double as[4], bs[4];
  int na = cut_span(r->a0, r->a1, oa.lo, oa.hi, as);
  int nb = cut_span(r->b0, r->b1, ob.lo, ob.hi, bs);
  int n = 0;
  for (int i = 0; i < na; ++i)
    for (int j = 0; j < nb; ++j) {
      out[n] = *r;
      out[n].a0 = as[i];
      out[n].a1 = as[i + 1];
      out[n].b0 = bs[j];
      out[n].b1 = bs[j + 1];
      ++n;
    }
  return n;
}

double orc_oracle_pair_integral(const orc_rect* Ii, const orc_rect* Ij, int depth) {
  /* oracle_pair_integral, SingleLayer branch (oracle.hpp:191-198) */
  if (same_geometry(Ii, Ij)) return rec_u(Ii, Ij, depth);
  orc_rect p1[9], p2[9];
  int n1 = presplit(Ii, Ij, p1), n2 = presplit(Ij, Ii, p2);
  double acc = 0.0;
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n2; ++j) acc += rec_u(&p1[i], &p2[j], depth);
  return acc;
}

/* ---------------- batch drivers ---------------- */

typedef struct {
  int64_t begin, end;
  const orc_rect *a, *b;
  double rel_tol;
  int max_levels;
  double* out;
  int* conv;
  int status;
} pair_job;

static void* pair_worker(void* vj) {
  pair_job* j = (pair_job*)vj;
  for (int64_t k = j->begin; k < j->end; ++k) {
    orc_kv kv = orc_u_pair_integral(&j->a[k], &j->b[k], j->rel_tol, j->max_levels);
    j->out[k] = kv.value;
    if (j->conv) j->conv[k] = kv.converged;
    if (kv.status) j->status = kv.status;
  }
  return NULL;
}

int orc_u_pairs(int64_t npairs, const orc_rect* a, const orc_rect* b, double rel_tol,
                int max_levels, double* out, int* converged, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  pair_job jobs[256];
  int64_t chunk = (npairs + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    jobs[t].begin = t * chunk < npairs ? t * chunk : npairs;
    jobs[t].end = (t + 1) * chunk < npairs ? (t + 1) * chunk : npairs;
    jobs[t].a = a;
    jobs[t].b = b;
    jobs[t].rel_tol = rel_tol;
    jobs[t].max_levels = max_levels;
    jobs[t].out = out;
    jobs[t].conv = converged;
    jobs[t].status = 0;
    if (nthreads == 1)
      pair_worker(&jobs[t]);
    else
      pthread_create(&th[t], NULL, pair_worker, &jobs[t]);
  }
  int status = 0;
  for (int t = 0; t < nthreads; ++t) {
    if (nthreads > 1) pthread_join(th[t], NULL);
    if (jobs[t].status) status = jobs[t].status;
  }
  return status;
}

typedef struct {
  int64_t n;
  const orc_rect* p;
  double rel_tol;
  int max_levels;
  double* A;
  int tid, nthreads;
  int all_conv, status;
} asm_job;

static void* asm_worker(void* vj) {
  asm_job* j = (asm_job*)vj;
  /* assemble_single loop (assembly.hpp:88-102); rows dealt round-robin */
  for (int64_t i = j->tid; i < j->n; i += j->nthreads) {
    double ai = (j->p[i].a1 - j->p[i].a0) * (j->p[i].b1 - j->p[i].b0);
    for (int64_t k = i; k < j->n; ++k) {
      orc_kv kv = orc_u_pair_integral(&j->p[i], &j->p[k], j->rel_tol, j->max_levels);
      if (kv.status) j->status = kv.status;
      if (!kv.converged) j->all_conv = 0;
      double ak = (j->p[k].a1 - j->p[k].a0) * (j->p[k].b1 - j->p[k].b0);
      double v = kv.value / (ai * ak);
      j->A[i * j->n + k] = v;
      j->A[k * j->n + i] = v;
    }
  }
  return NULL;
}

int orc_assemble_single(int64_t n, const orc_rect* p, double rel_tol, int max_levels,
                        double* A, int* all_converged, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  asm_job jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    asm_job j = {n, p, rel_tol, max_levels, A, t, nthreads, 1, 0};
    jobs[t] = j;
    if (nthreads == 1)
      asm_worker(&jobs[t]);
    else
      pthread_create(&th[t], NULL, asm_worker, &jobs[t]);
  }
  int status = 0, conv = 1;
  for (int t = 0; t < nthreads; ++t) {
    if (nthreads > 1) pthread_join(th[t], NULL);
    if (jobs[t].status) status = jobs[t].status;
    if (!jobs[t].all_conv) conv = 0;
  }
  if (all_converged) *all_converged = conv;
  return status;
}

/* ---------------- Cholesky factor in the reference's storage order ----------------
 * solver.hpp:28-37 with L an Eigen::MatrixXd, i.e. COLUMN-major: L(r, k) at
 * L[k * n + r], so L.row(k).head(k) walks with stride n (what the reference's
 * CPU loop actually does; the row-major restatement below is the fast
 * variant).  A is column-major too (symmetric, so either).  Timing only: returns
 * 0, or 2 with *bad_pivot on a non-positive pivot. */
int orc_cholesky_factor_colmajor(int64_t n, const double* A, double* L, int64_t* bad_pivot) {
  for (int64_t e = 0; e < n * n; ++e) L[e] = 0.0;
  for (int64_t k = 0; k < n; ++k) {
    double sq = 0.0;
    for (int64_t t = 0; t < k; ++t) sq += L[t * n + k] * L[t * n + k];
    double d = A[k * n + k] - sq;
    if (!(d > 0.0)) {
      if (bad_pivot) *bad_pivot = k;
      return 2;
    }
    L[k * n + k] = sqrt(d);
    for (int64_t r = k + 1; r < n; ++r) {
      double dot = 0.0;
      for (int64_t t = 0; t < k; ++t) dot += L[t * n + r] * L[t * n + k];
      L[k * n + r] = (A[k * n + r] - dot) / L[k * n + k];
    }
  }
  return 0;
}

/* ---------------- Cholesky (solver.hpp:17-50) ---------------- */

int orc_cholesky_solve(int64_t n, const double* A, int64_t nrhs, const double* B, double* X,
                       double* resid, int64_t* bad_pivot) {
  if (n < 0 || nrhs < 0) return 1;
  /* L stored row-major, lower triangle; reference loop order (solver.hpp:28-37) */
  double* L = (double*)calloc((size_t)(n > 0 ? n * n : 1), sizeof(double));
  if (!L) return 3;
  for (int64_t k = 0; k < n; ++k) {
    double sq = 0.0;
    for (int64_t t = 0; t < k; ++t) sq += L[k * n + t] * L[k * n + t];
    double d = A[k * n + k] - sq;
    if (!(d > 0.0)) {
      if (bad_pivot) *bad_pivot = k;
      free(L);
      return 2;
    }
    L[k * n + k] = sqrt(d);
    for (int64_t r = k + 1; r < n; ++r) {
      double dot = 0.0;
      for (int64_t t = 0; t < k; ++t) dot += L[r * n + t] * L[k * n + t];
      L[r * n + k] = (A[r * n + k] - dot) / L[k * n + k];
    }
  }
  double* y = (double*)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
  for (int64_t c = 0; c < nrhs; ++c) {
    const double* b = B + c * n;
    double* x = X + c * n;
    /* forward / back substitution (solver.hpp:39-44) */
    for (int64_t i = 0; i < n; ++i) {
      double s = 0.0;
      for (int64_t t = 0; t < i; ++t) s += L[i * n + t] * y[t];
      y[i] = (b[i] - s) / L[i * n + i];
    }
    for (int64_t i = n - 1; i >= 0; --i) {
      double s = 0.0;
      for (int64_t t = i + 1; t < n; ++t) s += L[t * n + i] * x[t];
      x[i] = (y[i] - s) / L[i * n + i];
    }
    if (resid) {
      /* residual_norm (solver.hpp:17-21) */
      double rn = 0.0, bn = 0.0;
      for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t t = 0; t < n; ++t) s += A[i * n + t] * x[t];
        rn += (s - b[i]) * (s - b[i]);
        bn += b[i] * b[i];
      }
      bn = sqrt(bn);
      resid[c] = sqrt(rn) / (bn > 0.0 ? bn : 1.0);
    }
  }
  free(y);
  free(L);
  return 0;
}

/* ---------------- point kernels (kernels.hpp:319-355) ---------------- */

static void inplane_axes(int axis, int* i0, int* i1) {
  *i0 = axis == 0 ? 1 : 0;
  *i1 = axis == 2 ? 1 : 2;
}

static double pt_F(double u, double v, double h, double h2, double guard) {
  double t = mul_log(v, u, v * v + h2, guard) + mul_log(u, v, u * u + h2, guard);
  if (h != 0.0) {
    double r = sqrt(u * u + v * v + h2);
    t -= h * atan(u * v / (h * r));
  }
  return t;
}

double orc_u_point_rect(const double x[3], const orc_rect* R) {
  int i0, i1;
  inplane_axes(R->axis, &i0, &i1);
  double h = x[R->axis] - R->level;
  double u1 = R->a0 - x[i0], u2 = R->a1 - x[i0];
  double v1 = R->b0 - x[i1], v2 = R->b1 - x[i1];
  double scale = fmax(fmax(fmax(fabs(u1), fabs(u2)), fmax(fabs(v1), fabs(v2))), fmax(fabs(h), 1e-30));
  double guard = 1e-14 * scale, h2 = h * h;
  return (pt_F(u2, v2, h, h2, guard) - pt_F(u1, v2, h, h2, guard) - pt_F(u2, v1, h, h2, guard) +
          pt_F(u1, v1, h, h2, guard)) /
         kFourPi;
}

static double pt_G(double u, double v, double h, double h2) {
  double r = sqrt(u * u + v * v + h2);
  return atan(u * v / (h * r));
}

double orc_q_point_rect(const double x[3], const orc_rect* R, int nsign) {
  double h = x[R->axis] - R->level;
  if (h == 0.0) return 0.0;
  int i0, i1;
  inplane_axes(R->axis, &i0, &i1);
  double u1 = R->a0 - x[i0], u2 = R->a1 - x[i0];
  double v1 = R->b0 - x[i1], v2 = R->b1 - x[i1];
  double h2 = h * h;
  double sum = pt_G(u2, v2, h, h2) - pt_G(u1, v2, h, h2) - pt_G(u2, v1, h, h2) + pt_G(u1, v1, h, h2);
  return (double)nsign * sum / kFourPi;
}

/* ---------------- collocation block system (assembly.hpp:37-75,179-227) ---------------- */

int orc_assemble_collocation(int64_t n, const orc_rect* p, const int* nsign, const int* kind, const int* net,
                             const int* reg_a, const int* reg_b, int nreg, const int* reg_id,
                             const double* reg_eps, int main_net, double* A, double* b, int64_t* m_out) {
  int64_t off[5] = {0, 0, 0, 0, 0};
  for (int64_t k = 0; k < n; ++k) off[kind[k] + 1]++;
  for (int k = 1; k < 5; ++k) off[k] += off[k - 1];
  if (off[2] == 0) return 1; /* no conductor / Dirichlet panel */
  int64_t o3 = off[3];
  int64_t* qcol = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t* ucol = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t q = 0; q < n; ++q) { /* buildUnknownMap */
    qcol[q] = ucol[q] = -1;
    if (kind[q] == 0 || kind[q] == 1) qcol[q] = q;
    else if (kind[q] == 2) ucol[q] = q;
    else {
      ucol[q] = o3 + 2 * (q - o3);
      qcol[q] = o3 + 2 * (q - o3) + 1;
    }
  }
  int64_t cols = o3 + 2 * (off[4] - o3);
  /* regions in ascending id (std::map order) */
  int* order = (int*)malloc(sizeof(int) * (size_t)nreg);
  for (int k = 0; k < nreg; ++k) order[k] = k;
  for (int a = 0; a < nreg; ++a)
    for (int c = a + 1; c < nreg; ++c)
      if (reg_id[order[c]] < reg_id[order[a]]) {
        int t = order[a];
        order[a] = order[c];
        order[c] = t;
      }
  for (int64_t q = 0; q < n; ++q) {
    int found = 0;
    for (int k = 0; k < nreg; ++k) found |= reg_a[q] == reg_id[k];
    if (!found) {
      free(qcol); free(ucol); free(order);
      return 1;
    }
  }
  /* rows: per region (ascending), panels with regionA == id or interface with regionB == id */
  int64_t rows = 0;
  for (int k = 0; k < nreg; ++k) {
    int rid = reg_id[order[k]];
    for (int64_t q = 0; q < n; ++q)
      if (reg_a[q] == rid || (kind[q] == 3 && reg_b[q] == rid)) rows++;
  }
  if (rows != cols) {
    free(qcol); free(ucol); free(order);
    return 2;
  }
  int64_t m = rows;
  for (int64_t i = 0; i < m * m; ++i) A[i] = 0.0;
  for (int64_t i = 0; i < m; ++i) b[i] = 0.0;
  int64_t row = 0;
  for (int k = 0; k < nreg; ++k) {
    int rid = reg_id[order[k]];
    double eps_r = reg_eps[order[k]];
    for (int64_t a = 0; a < n; ++a) {
      if (!(reg_a[a] == rid || (kind[a] == 3 && reg_b[a] == rid))) continue;
      double x[3];
      for (int d = 0; d < 3; ++d) {
        span_t e = rect_extent(&p[a], d);
        x[d] = 0.5 * (e.lo + e.hi); /* Rect::center */
      }
      for (int64_t c = 0; c < n; ++c) {
        if (!(reg_a[c] == rid || (kind[c] == 3 && reg_b[c] == rid))) continue;
        double side = kind[c] == 3 ? (reg_a[c] == rid ? 1.0 : -1.0) : -1.0; /* sideSign */
        double coefU = orc_q_point_rect(x, &p[c], nsign[c]) * side + (a == c ? 0.5 : 0.0);
        double known = (kind[c] == 0 && net[c] == main_net) ? 1.0 : 0.0; /* knownPotential */
        if (ucol[c] >= 0)
          A[row * m + ucol[c]] += coefU;
        else
          b[row] -= coefU * known;
        if (kind[c] == 2) continue;
        double area = (p[c].a1 - p[c].a0) * (p[c].b1 - p[c].b0);
        double coefX = -orc_u_point_rect(x, &p[c]) / area;
        if (kind[c] == 3 && reg_b[c] == rid) {
          double eps_a = 1.0;
          for (int t = 0; t < nreg; ++t)
            if (reg_id[t] == reg_a[c]) eps_a = reg_eps[t];
          coefX *= -(eps_a / eps_r);
        }
        A[row * m + qcol[c]] += coefX;
      }
      row++;
    }
  }
  free(qcol);
  free(ucol);
  free(order);
  if (m_out) *m_out = m;
  return 0;
}

/* ---------------- Galerkin block system (assembly.hpp:37-75, 110-175) ---------------- */

int orc_assemble_multi(int64_t n, const orc_rect* p, const int* nsign, const int* kind, const int* net,
                       const int* reg_a, const int* reg_b, int nreg, const int* reg_id, const double* reg_eps,
                       int main_net, double rel_tol, int max_levels, double* A, double* b, int64_t* m_out,
                       int* all_converged) {
  int64_t off[5] = {0, 0, 0, 0, 0};
  for (int64_t k = 0; k < n; ++k) off[kind[k] + 1]++;
  for (int k = 1; k < 5; ++k) off[k] += off[k - 1];
  if (off[2] == 0) return 1;
  int64_t o3 = off[3];
  int64_t* qcol = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t* ucol = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t q = 0; q < n; ++q) { /* buildUnknownMap (assembly.hpp:51-75) */
    qcol[q] = ucol[q] = -1;
    if (kind[q] == 0 || kind[q] == 1) qcol[q] = q;
    else if (kind[q] == 2) ucol[q] = q;
    else {
      ucol[q] = o3 + 2 * (q - o3);
      qcol[q] = o3 + 2 * (q - o3) + 1;
    }
  }
  int64_t cols = o3 + 2 * (off[4] - o3);
  int* order = (int*)malloc(sizeof(int) * (size_t)nreg);
  for (int k = 0; k < nreg; ++k) order[k] = k;
  for (int a = 0; a < nreg; ++a)
    for (int c = a + 1; c < nreg; ++c)
      if (reg_id[order[c]] < reg_id[order[a]]) {
        int t = order[a];
        order[a] = order[c];
        order[c] = t;
      }
  for (int64_t q = 0; q < n; ++q) {
    int found = 0;
    for (int k = 0; k < nreg; ++k) found |= reg_a[q] == reg_id[k];
    if (!found) {
      free(qcol); free(ucol); free(order);
      return 1;
    }
  }
  int64_t rows = 0;
  for (int k = 0; k < nreg; ++k) {
    int rid = reg_id[order[k]];
    for (int64_t q = 0; q < n; ++q)
      if (reg_a[q] == rid || (kind[q] == 3 && reg_b[q] == rid)) rows++;
  }
  if (rows != cols) {
    free(qcol); free(ucol); free(order);
    return 2;
  }
  int64_t m = rows;
  for (int64_t i = 0; i < m * m; ++i) A[i] = 0.0;
  for (int64_t i = 0; i < m; ++i) b[i] = 0.0;
  int conv = 1;
  int64_t row = 0;
  for (int k = 0; k < nreg; ++k) {
    int rid = reg_id[order[k]];
    double eps_r = reg_eps[order[k]];
    for (int64_t a = 0; a < n; ++a) {
      if (!(reg_a[a] == rid || (kind[a] == 3 && reg_b[a] == rid))) continue;
      double area_a = (p[a].a1 - p[a].a0) * (p[a].b1 - p[a].b0);
      for (int64_t c = 0; c < n; ++c) {
        if (!(reg_a[c] == rid || (kind[c] == 3 && reg_b[c] == rid))) continue;
        /* Qloc(a, c) = q_pair_integral(P_a, P_c) * sideSign(P_c, region) */
        orc_kv kq = orc_q_pair_integral(&p[a], &p[c], nsign[c], rel_tol, max_levels);
        if (kq.status) { free(qcol); free(ucol); free(order); return 3; }
        conv &= kq.converged;
        double side = kind[c] == 3 ? (reg_a[c] == rid ? 1.0 : -1.0) : -1.0; /* sideSign (assembly.hpp:37-40) */
        double coefU = kq.value * side / area_a + (a == c ? 0.5 : 0.0);
        double known = (kind[c] == 0 && net[c] == main_net) ? 1.0 : 0.0; /* knownPotential */
        if (ucol[c] >= 0)
          A[row * m + ucol[c]] += coefU;
        else
          b[row] -= coefU * known;
        if (kind[c] == 2) continue;
        orc_kv ku = orc_u_pair_integral(&p[a], &p[c], rel_tol, max_levels);
        if (ku.status) { free(qcol); free(ucol); free(order); return 3; }
        conv &= ku.converged;
        double area_c = (p[c].a1 - p[c].a0) * (p[c].b1 - p[c].b0);
        double coefX = -ku.value / (area_a * area_c);
        if (kind[c] == 3 && reg_b[c] == rid) {
          double eps_a = 1.0;
          for (int t = 0; t < nreg; ++t)
            if (reg_id[t] == reg_a[c]) eps_a = reg_eps[t];
          coefX *= -(eps_a / eps_r);
        }
        A[row * m + qcol[c]] += coefX;
      }
      row++;
    }
  }
  free(qcol);
  free(ucol);
  free(order);
  if (m_out) *m_out = m;
  if (all_converged) *all_converged = conv;
  return 0;
}

/* ---------------- LU with partial pivoting (solver.hpp:53-88) ---------------- */

int orc_lu_solve(int64_t n, const double* A0, const double* b0, double* x, double* resid, int64_t* bad_row) {
  double* A = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n * n : 1));
  double* b = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  memcpy(A, A0, sizeof(double) * (size_t)(n * n));
  memcpy(b, b0, sizeof(double) * (size_t)n);
  double scale = 0.0;
  for (int64_t i = 0; i < n * n; ++i) scale = fmax(scale, fabs(A[i]));
  for (int64_t k = 0; k < n; ++k) {
    int64_t pr = k; /* first maximum, as Eigen's maxCoeff */
    double best = fabs(A[k * n + k]);
    for (int64_t r = k + 1; r < n; ++r)
      if (fabs(A[r * n + k]) > best) {
        best = fabs(A[r * n + k]);
        pr = r;
      }
    if (pr != k) {
      for (int64_t c = 0; c < n; ++c) {
        double t = A[k * n + c];
        A[k * n + c] = A[pr * n + c];
        A[pr * n + c] = t;
      }
      double t = b[k];
      b[k] = b[pr];
      b[pr] = t;
    }
    if (fabs(A[k * n + k]) < 1e-14 * scale) {
      if (bad_row) *bad_row = k;
      free(A);
      free(b);
      return 2;
    }
    for (int64_t r = k + 1; r < n; ++r) {
      double f = A[r * n + k] / A[k * n + k];
      if (f == 0.0) continue;
      for (int64_t c = k + 1; c < n; ++c) A[r * n + c] -= f * A[k * n + c];
      b[r] -= f * b[k];
    }
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    double s = 0.0;
    for (int64_t t = i + 1; t < n; ++t) s += A[i * n + t] * x[t];
    x[i] = (b[i] - s) / A[i * n + i];
  }
  if (resid) {
    double rn = 0.0, bn = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double s = 0.0;
      for (int64_t t = 0; t < n; ++t) s += A0[i * n + t] * x[t];
      rn += (s - b0[i]) * (s - b0[i]);
      bn += b0[i] * b0[i];
    }
    bn = sqrt(bn);
    *resid = sqrt(rn) / (bn > 0.0 ? bn : 1.0);
  }
  free(A);
  free(b);
  return 0;
}

/* ---------------- quadrature known-answer hooks ---------------- */

static double qt_f(const void* vc, double x) {
  int which = *(const int*)vc;
  switch (which) {
    case 0: return x * x;
    case 1: return 1.0;
    case 2: return log1p(x);
    case 3: return x;
    case 4: return sin(x);
    case 5: return 1.0 / x;
    case 6: return 1.0 / sqrt(x);
    case 7: return log(x);
    case 8: return 1.0 / sqrt(1.0 - x);
    case 9: return 1.0 / sqrt(x) + 1.0 / sqrt(1.0 - x);
    case 10: return 1.0 / sqrt(fabs(x));
    default: return x * x;
  }
}

double orc_quad_test(int which, int mode, double a, double b, int singA, int singB,
                     int* status, int* converged, long* evals) {
  qstats st = {0, 1, 0};
  double v;
  if (mode == 0)
    v = romberg(qt_f, &which, a, b, 1e-8, 16, &st);
  else if (mode == 1)
    v = integrate_segment(qt_f, &which, a, b, singA, singB, 1e-8, 16, &st);
  else
    v = integrate_with_splits(qt_f, &which, a, b, 1e-8, 16, &st);
  if (status) *status = st.status;
  if (converged) *converged = st.converged;
  if (evals) *evals = st.evals;
  return v;
}

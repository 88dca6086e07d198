/* Experiment: replace the reference's adaptive Romberg (quadrature.hpp:27-64)
 * on the reduced 1-D integrands by a fixed rule: every reference segment is
 * split at its midpoint and each half is integrated with the t^POW endpoint
 * substitution toward its outer end and an n-point Gauss-Legendre rule in t.
 * Compares against the tight-tolerance reference algorithm (relTol 1e-14). */
#include "../oracle/gbem_oracle.c"
#include <stdio.h>

static double GLX[65][64], GLW[65][64];
static void gl_init(void) {
  for (int n = 1; n <= 64; ++n)
    for (int i = 0; i < n; ++i) {
      double x = cos(M_PI * (i + 0.75) / (n + 0.5));
      for (int it = 0; it < 100; ++it) {
        double p0 = 1, p1 = x;
        for (int k = 2; k <= n; ++k) { double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k; p0 = p1; p1 = p2; }
        double dp = n * (x * p1 - p0) / (x * x - 1);
        double dx = p1 / dp; x -= dx;
        if (fabs(dx) < 1e-16) break;
      }
      double p0 = 1, p1 = x;
      for (int k = 2; k <= n; ++k) { double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k; p0 = p1; p1 = p2; }
      double dp = n * (x * p1 - p0) / (x * x - 1);
      GLX[n][i] = x; GLW[n][i] = 2 / ((1 - x * x) * dp * dp);
    }
}
static int NG = 16, POW = 4;
static double gl_graded(integrand_fn f, const void* ctx, double a, double b) {
  if (a == b) return 0.0;
  double m = 0.5 * (a + b), total = 0.0;
  for (int side = 0; side < 2; ++side) {
    double base = side ? b : a, len = side ? b - m : m - a;
    double T = pow(len, 1.0 / POW), h = 0.5 * T;
    for (int i = 0; i < NG; ++i) {
      double t = h + h * GLX[NG][i];
      double tp = pow(t, POW - 1);
      double x = side ? base - tp * t : base + tp * t;
      total += h * GLW[NG][i] * POW * tp * f(ctx, x);
    }
  }
  return total;
}
static double gl_par(span_t sx, span_t sy, span_t tx, span_t ty, double b) {
  par_ctx c; c.b2 = b * b;
  u_corners(sx.lo, sx.hi, tx.lo, tx.hi, c.sign, c.val);
  double cuts[5]; int count = tent_segments(sy.lo, sy.hi, ty.lo, ty.hi, &c.w, cuts);
  double total = 0.0;
  for (int i = 0; i + 1 < count; ++i) total += gl_graded(par_f, &c, cuts[i], cuts[i + 1]);
  return total / kFourPi;
}
static double gl_split0(integrand_fn f, const void* ctx, double a, double b) {
  if (a < 0.0 && 0.0 < b) return gl_graded(f, ctx, a, 0.0) + gl_graded(f, ctx, 0.0, b);
  return gl_graded(f, ctx, a, b);
}
static double gl_orth(span_t s1, span_t s3, span_t t1, span_t t2) {
  orth_ctx c;
  u_corners(s1.lo, s1.hi, t1.lo, t1.hi, c.sign, c.val);
  c.x3d = s3.lo; c.x3u = s3.hi; c.y2d = t2.lo; c.y2u = t2.hi;
  double scale = max4(s1.hi - s1.lo, t1.hi - t1.lo, s3.hi - s3.lo, t2.hi - t2.lo);
  if (scale < 1e-30) scale = 1e-30;
  c.guard = 1e-14 * scale;
  return (gl_split0(orth_fx, &c, c.x3d, c.x3u) + gl_split0(orth_fy, &c, t2.lo, t2.hi)) / kFourPi;
}
static double gl_pair(const orc_rect* Ii, const orc_rect* Ij) {
  const orc_rect* a = rect_less(Ij, Ii) ? Ij : Ii;
  const orc_rect* b = rect_less(Ij, Ii) ? Ii : Ij;
  span_t aA = {a->a0, a->a1}, aB = {a->b0, a->b1}, bA = {b->a0, b->a1}, bB = {b->b0, b->b1};
  if (a->axis == b->axis) {
    double off = a->level - b->level;
    if (off == 0.0) return u_coplanar(aA, aB, bA, bB);
    return gl_par(aA, aB, bA, bB, off);
  }
  int shared = 3 - a->axis - b->axis;
  span_t s1 = rect_extent(a, shared), t1 = rect_extent(b, shared);
  span_t i3 = rect_extent(a, b->axis), j2 = rect_extent(b, a->axis);
  span_t s3 = {i3.lo - b->level, i3.hi - b->level}, t2 = {j2.lo - a->level, j2.hi - a->level};
  return gl_orth(s1, s3, t1, t2);
}
int main(int argc, char** argv) {
  gl_init();
  FILE* f = fopen(argv[1], "r");
  int n;
  if (fscanf(f, "%d", &n) != 1) return 1;
  orc_rect* A = malloc(sizeof(orc_rect) * n);
  orc_rect* B = malloc(sizeof(orc_rect) * n);
  double* g = malloc(sizeof(double) * n);
  for (int k = 0; k < n; ++k) {
    if (fscanf(f, "%d %lf %lf %lf %lf %lf", &A[k].axis, &A[k].level, &A[k].a0, &A[k].a1, &A[k].b0, &A[k].b1) != 6) return 1;
    if (fscanf(f, "%d %lf %lf %lf %lf %lf %lf", &B[k].axis, &B[k].level, &B[k].a0, &B[k].a1, &B[k].b0, &B[k].b1, &g[k]) != 7) return 1;
  }
  double* tight = malloc(sizeof(double) * n);
  double worst_ref = 0;
  for (int k = 0; k < n; ++k) {
    orc_kv t = orc_u_pair_integral(&A[k], &B[k], 1e-14, 24);
    orc_kv r = orc_u_pair_integral(&A[k], &B[k], 1e-8, 16);
    tight[k] = t.value;
    double er = fabs(r.value - t.value) / fabs(t.value);
    if (er > worst_ref) worst_ref = er;
  }
  printf("reference (relTol 1e-8) vs tight: worst %.2e\n", worst_ref);
  int ns[] = {8, 12, 16, 20, 24, 32, 48};
  for (int pw = 2; pw <= 4; ++pw) {
    POW = pw;
    for (int q = 0; q < 7; ++q) {
      NG = ns[q];
      double worst = 0, worst_touch = 0;
      int wk = -1;
      for (int k = 0; k < n; ++k) {
        double v = gl_pair(&A[k], &B[k]);
        double e = fabs(v - tight[k]) / fabs(tight[k]);
        if (g[k] == 0.0) { if (e > worst_touch) worst_touch = e; }
        else if (e > worst) { worst = e; wk = k; }
      }
      printf("pow=%d n=%2d worst_nontouch=%.2e (g=%.3g) worst_touch=%.2e\n", POW, NG, worst,
             wk >= 0 ? g[wk] : -1, worst_touch);
    }
  }
  return 0;
}

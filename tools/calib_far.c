/* Calibrate the anisotropic far-field tensor-Gauss order rule.
 * For a direction of half-length h at gap d from the other panel, delta = d/h
 * and the Bernstein-ellipse radius of the end-on singularity is
 * rho = 1 + delta + sqrt(delta*(2+delta)); the q-point Gauss error of that
 * direction behaves like C*rho^(-2q).  We pick q_k = min q with
 * rho^(-2q) <= tol_dir, then measure the true relative error of the product
 * rule over seeded random pairs vs a composite high-order truth. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>

typedef struct { int axis; double level, a0, a1, b0, b1; } rect;
static double GX[17][16], GW[17][16];
static void legendre_init(void) {
  for (int n = 1; n <= 16; ++n) {
    for (int i = 0; i < n; ++i) {
      double x = cos(M_PI * (i + 0.75) / (n + 0.5));
      for (int it = 0; it < 100; ++it) {
        double p0 = 1, p1 = x;
        for (int k = 2; k <= n; ++k) { double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k; p0 = p1; p1 = p2; }
        if (n == 1) { p1 = x; p0 = 1; }
        double dp = n * (x * p1 - p0) / (x * x - 1);
        double dx = p1 / dp; x -= dx; if (fabs(dx) < 1e-17) break;
      }
      double p0 = 1, p1 = x;
      for (int k = 2; k <= n; ++k) { double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k; p0 = p1; p1 = p2; }
      double dp = n * (x * p1 - p0) / (x * x - 1);
      GX[n][i] = -x; GW[n][i] = 2 / ((1 - x * x) * dp * dp);
    }
  }
}
static void ip(int axis, int* i0, int* i1) { *i0 = axis == 0 ? 1 : 0; *i1 = axis == 2 ? 1 : 2; }
static double gauss4(const rect* P, const rect* Q, int qs, int qt, int qu, int qv) {
  int p0, p1, q0, q1; ip(P->axis, &p0, &p1); ip(Q->axis, &q0, &q1);
  double acc = 0;
  for (int s = 0; s < qs; ++s) for (int t = 0; t < qt; ++t) {
    double x[3]; x[P->axis] = P->level;
    double ha = 0.5 * (P->a1 - P->a0), hb = 0.5 * (P->b1 - P->b0);
    x[p0] = 0.5 * (P->a0 + P->a1) + ha * GX[qs][s]; x[p1] = 0.5 * (P->b0 + P->b1) + hb * GX[qt][t];
    double w1 = ha * GW[qs][s] * hb * GW[qt][t];
    for (int u = 0; u < qu; ++u) for (int v = 0; v < qv; ++v) {
      double y[3]; y[Q->axis] = Q->level;
      double hc = 0.5 * (Q->a1 - Q->a0), hd = 0.5 * (Q->b1 - Q->b0);
      y[q0] = 0.5 * (Q->a0 + Q->a1) + hc * GX[qu][u]; y[q1] = 0.5 * (Q->b0 + Q->b1) + hd * GX[qv][v];
      double w2 = hc * GW[qu][u] * hd * GW[qv][v];
      double dx = x[0] - y[0], dy = x[1] - y[1], dz = x[2] - y[2];
      acc += w1 * w2 / sqrt(dx * dx + dy * dy + dz * dz);
    }
  }
  return acc / (4 * M_PI);
}
static double truth(const rect* P, const rect* Q) {
  int S = 3; double acc = 0;
  for (int i = 0; i < S; ++i) for (int j = 0; j < S; ++j) for (int k = 0; k < S; ++k) for (int l = 0; l < S; ++l) {
    rect a = *P, b = *Q;
    a.a0 = P->a0 + (P->a1 - P->a0) * i / S; a.a1 = P->a0 + (P->a1 - P->a0) * (i + 1) / S;
    a.b0 = P->b0 + (P->b1 - P->b0) * j / S; a.b1 = P->b0 + (P->b1 - P->b0) * (j + 1) / S;
    b.a0 = Q->a0 + (Q->a1 - Q->a0) * k / S; b.a1 = Q->a0 + (Q->a1 - Q->a0) * (k + 1) / S;
    b.b0 = Q->b0 + (Q->b1 - Q->b0) * l / S; b.b1 = Q->b0 + (Q->b1 - Q->b0) * (l + 1) / S;
    acc += gauss4(&a, &b, 12, 12, 12, 12);
  }
  return acc;
}
static void ext(const rect* r, int k, double* lo, double* hi) {
  int i0, i1; ip(r->axis, &i0, &i1);
  if (k == r->axis) { *lo = *hi = r->level; } else if (k == i0) { *lo = r->a0; *hi = r->a1; } else { *lo = r->b0; *hi = r->b1; }
}
static double gap(const rect* a, const rect* b) {
  double s = 0;
  for (int k = 0; k < 3; ++k) { double la, ha, lb, hb; ext(a, k, &la, &ha); ext(b, k, &lb, &hb);
    double g = fmax(fmax(lb - ha, la - hb), 0); s += g * g; }
  return sqrt(s);
}
static double diam(const rect* r) { return hypot(r->a1 - r->a0, r->b1 - r->b0); }
static uint64_t st = 88172645463325252ull;
static double U(void) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return (st >> 11) * (1.0 / 9007199254740992.0); }
static int qfor(double h, double d, double logtol) {
  double del = d / h; double rho = 1 + del + sqrt(del * (2 + del));
  int q = (int)ceil(logtol / (-2 * log(rho)));
  if (q < 1) q = 1; if (q > 16) q = 16; return q;
}
int main(int argc, char** argv) {
  legendre_init();
  double tol = argc > 1 ? atof(argv[1]) : 1e-13;
  double logtol = log(tol);
  double gs[] = {0.5, 0.75, 1, 1.5, 2, 3, 4, 6, 8, 12, 16, 32, 64};
  for (int gi = 0; gi < 13; ++gi) {
    double worst = 0, sumev = 0; int N = 400, over = 0;
    for (int n = 0; n < N; ++n) {
      rect P, Q;
      P.axis = (int)(U() * 3); P.level = 0;
      double la = 0.2 + U(), asp = U() < 0.5 ? 1 : exp((U() * 2 - 1) * log(10.0)), lb = la * asp;
      P.a0 = -la / 2; P.a1 = la / 2; P.b0 = -lb / 2; P.b1 = lb / 2;
      int cls = (int)(U() * 3);
      Q.axis = cls < 2 ? P.axis : (P.axis + 1 + (int)(U() * 2)) % 3;
      double s = exp((U() * 2 - 1) * log(8.0));
      double lc = (0.2 + U()) * s, asp2 = U() < 0.5 ? 1 : exp((U() * 2 - 1) * log(10.0)), ld = lc * asp2;
      double d[3] = {U() * 2 - 1, U() * 2 - 1, U() * 2 - 1};
      if (cls == 0) d[P.axis] = 0;
      double nn = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]); for (int k = 0; k < 3; ++k) d[k] /= nn;
      double dm = fmax(diam(&P), hypot(lc, ld));
      double lo = 0, hi = 200;
      for (int it = 0; it < 80; ++it) {
        double m = 0.5 * (lo + hi); int q0, q1; ip(Q.axis, &q0, &q1);
        Q.level = cls == 0 ? 0 : d[Q.axis] * m;
        Q.a0 = d[q0] * m - lc / 2; Q.a1 = d[q0] * m + lc / 2; Q.b0 = d[q1] * m - ld / 2; Q.b1 = d[q1] * m + ld / 2;
        if (gap(&P, &Q) / dm < gs[gi]) lo = m; else hi = m;
      }
      double gp = gap(&P, &Q);
      int qs = qfor(0.5 * (P.a1 - P.a0), gp, logtol), qt = qfor(0.5 * (P.b1 - P.b0), gp, logtol);
      int qu = qfor(0.5 * (Q.a1 - Q.a0), gp, logtol), qv = qfor(0.5 * (Q.b1 - Q.b0), gp, logtol);
      double v = gauss4(&P, &Q, qs, qt, qu, qv), tr = truth(&P, &Q);
      double e = fabs(v - tr) / tr; if (e > worst) worst = e; if (e > 1e-11) over++;
      sumev += qs * qt * qu * qv;
    }
    printf("g=%5.2f worst=%.2e mean_evals=%.0f over1e-11=%d\n", gs[gi], worst, sumev / N, over);
    fflush(stdout);
  }
}

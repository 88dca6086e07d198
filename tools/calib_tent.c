/* Calibrate the difference-set ("tent") far-field rule against a composite
 * high-order truth.  For a shared in-plane axis of two panels with spans
 * [s0,s1] and [u0,u1], the x - y difference w has the trapezoidal density
 * T(w) = |[s0,s1] ∩ [u0+w,u1+w]| (ramp, plateau, ramp), so the 4-D integral
 * becomes a 2-D (parallel) or 3-D (orthogonal) one with piecewise-linear
 * weights; each piece gets Gauss-Legendre of the order the far-field rule gives
 * its half-length at the pair's gap.  Per axis the cheaper of the tent and the
 * plain product rule (q_i q_j nodes) is used.  Prints worst relative error and
 * mean node counts per gap/diameter ratio.
 *   cc -O2 -o /tmp/calib_tent tools/calib_tent.c -lm && /tmp/calib_tent [tol=1e-12] [pairs=200] */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

typedef struct { int axis; double level, a0, a1, b0, b1; } rect;
static double GX[17][16], GW[17][16];
static void legendre_init(void) {
  for (int n = 1; n <= 16; ++n)
    for (int i = 0; i < n; ++i) {
      double x = cos(M_PI * (i + 0.75) / (n + 0.5));
      for (int it = 0; it < 100; ++it) {
        double p0 = 1, p1 = x;
        for (int k = 2; k <= n; ++k) { double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k; p0 = p1; p1 = p2; }
        if (n == 1) { p1 = x; p0 = 1; }
        double dp = n * (x * p1 - p0) / (x * x - 1), dx = p1 / dp;
        x -= dx;
        if (fabs(dx) < 1e-17) break;
      }
      double p0 = 1, p1 = x;
      for (int k = 2; k <= n; ++k) { double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k; p0 = p1; p1 = p2; }
      if (n == 1) { p1 = x; p0 = 1; }
      double dp = n * (x * p1 - p0) / (x * x - 1);
      GX[n][i] = -x; GW[n][i] = 2 / ((1 - x * x) * dp * dp);
    }
}
static void ip(int axis, int* i0, int* i1) { *i0 = axis == 0 ? 1 : 0; *i1 = axis == 2 ? 1 : 2; }
static void ext(const rect* r, int k, double* lo, double* hi) {
  int i0, i1; ip(r->axis, &i0, &i1);
  if (k == r->axis) { *lo = *hi = r->level; } else if (k == i0) { *lo = r->a0; *hi = r->a1; } else { *lo = r->b0; *hi = r->b1; }
}
static double gauss4(const rect* P, const rect* Q, int qs, int qt, int qu, int qv) {
  int p0, p1, q0, q1; ip(P->axis, &p0, &p1); ip(Q->axis, &q0, &q1);
  double acc = 0, ha = 0.5 * (P->a1 - P->a0), hb = 0.5 * (P->b1 - P->b0);
  double hc = 0.5 * (Q->a1 - Q->a0), hd = 0.5 * (Q->b1 - Q->b0);
  for (int s = 0; s < qs; ++s) for (int t = 0; t < qt; ++t) {
    double x[3]; x[P->axis] = P->level;
    x[p0] = 0.5 * (P->a0 + P->a1) + ha * GX[qs][s]; x[p1] = 0.5 * (P->b0 + P->b1) + hb * GX[qt][t];
    double w1 = ha * GW[qs][s] * hb * GW[qt][t];
    for (int u = 0; u < qu; ++u) for (int v = 0; v < qv; ++v) {
      double y[3]; y[Q->axis] = Q->level;
      y[q0] = 0.5 * (Q->a0 + Q->a1) + hc * GX[qu][u]; y[q1] = 0.5 * (Q->b0 + Q->b1) + hd * GX[qv][v];
      double dx = x[0] - y[0], dy = x[1] - y[1], dz = x[2] - y[2];
      acc += w1 * hc * GW[qu][u] * hd * GW[qv][v] / sqrt(dx * dx + dy * dy + dz * dz);
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
static double gap(const rect* a, const rect* b) {
  double s = 0;
  for (int k = 0; k < 3; ++k) {
    double la, ha, lb, hb; ext(a, k, &la, &ha); ext(b, k, &lb, &hb);
    double g = fmax(fmax(lb - ha, la - hb), 0); s += g * g;
  }
  return sqrt(s);
}
static double diam(const rect* r) { return hypot(r->a1 - r->a0, r->b1 - r->b0); }
static uint64_t st = 88172645463325252ull;
static double U(void) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return (st >> 11) * (1.0 / 9007199254740992.0); }

static double g_delta[17];
static int qfor(double h, double d) {  /* smallest q with d/h >= delta[q] */
  if (h <= 0) return 1;
  int q = 1;
  while (q < 16 && d / h < g_delta[q]) ++q;
  return q;
}
/* node list of one axis */
typedef struct { int m; double w[64], W[64]; } list;
static void add_gauss(list* L, double lo, double hi, int q, double wlo, double whi, double shift) {
  /* nodes of [lo,hi] (in w), weight density linear from wlo at lo to whi at hi */
  double c = 0.5 * (lo + hi), h = 0.5 * (hi - lo);
  for (int k = 0; k < q; ++k) {
    double x = c + h * GX[q][k], t = (x - lo) / (hi - lo);
    L->w[L->m] = x + shift;
    L->W[L->m] = h * GW[q][k] * (wlo + (whi - wlo) * t);
    L->m++;
  }
}
static int tent_choice = 1;  /* 0: product only, 1: min(product, tent) */
static void shared_list(list* L, double s0, double s1, double u0, double u1, double d) {
  double Li = s1 - s0, Lj = u1 - u0;
  int qi = qfor(0.5 * Li, d), qj = qfor(0.5 * Lj, d);
  double mn = fmin(Li, Lj), hp = 0.5 * fabs(Li - Lj);
  int qr = qfor(0.5 * mn, d), qp = hp > 1e-9 * mn ? qfor(hp, d) : 0;
  L->m = 0;
  if (!tent_choice || qi * qj <= 2 * qr + qp) {
    double ci = 0.5 * (s0 + s1), cj = 0.5 * (u0 + u1);
    for (int a = 0; a < qi; ++a) for (int b = 0; b < qj; ++b) {
      L->w[L->m] = (ci + 0.5 * Li * GX[qi][a]) - (cj + 0.5 * Lj * GX[qj][b]);
      L->W[L->m] = 0.5 * Li * GW[qi][a] * 0.5 * Lj * GW[qj][b];
      L->m++;
    }
    return;
  }
  double wl = s0 - u1, k1 = fmin(s0 - u0, s1 - u1), k2 = fmax(s0 - u0, s1 - u1), wh = s1 - u0;
  add_gauss(L, wl, k1, qr, 0.0, mn, 0);
  if (qp) add_gauss(L, k1, k2, qp, mn, mn, 0);
  add_gauss(L, k2, wh, qr, mn, 0.0, 0);
}
static void single_list(list* L, double lo, double hi, double d, double sign, double off) {
  /* w = sign * x - off for x in [lo, hi] */
  int q = qfor(0.5 * (hi - lo), d);
  L->m = 0;
  for (int k = 0; k < q; ++k) {
    double x = 0.5 * (lo + hi) + 0.5 * (hi - lo) * GX[q][k];
    L->w[L->m] = sign * x - off;
    L->W[L->m] = 0.5 * (hi - lo) * GW[q][k];
    L->m++;
  }
}
static double tent_rule(const rect* P, const rect* Q, long* nodes) {
  double d = gap(P, Q);
  list A, B, C;
  if (P->axis == Q->axis) {
    int k1, k2; ip(P->axis, &k1, &k2);
    double s0, s1, u0, u1;
    ext(P, k1, &s0, &s1); ext(Q, k1, &u0, &u1); shared_list(&A, s0, s1, u0, u1, d);
    ext(P, k2, &s0, &s1); ext(Q, k2, &u0, &u1); shared_list(&B, s0, s1, u0, u1, d);
    C.m = 1; C.w[0] = P->level - Q->level; C.W[0] = 1;
  } else {
    int k3 = 3 - P->axis - Q->axis;
    double s0, s1, u0, u1;
    ext(P, k3, &s0, &s1); ext(Q, k3, &u0, &u1); shared_list(&A, s0, s1, u0, u1, d);
    ext(P, Q->axis, &s0, &s1); single_list(&B, s0, s1, d, 1.0, Q->level);   /* x - Q.level */
    ext(Q, P->axis, &u0, &u1); single_list(&C, u0, u1, d, -1.0, -P->level); /* P.level - y */
  }
  double acc = 0;
  for (int a = 0; a < A.m; ++a) for (int b = 0; b < B.m; ++b) for (int c = 0; c < C.m; ++c)
    acc += A.W[a] * B.W[b] * C.W[c] / sqrt(A.w[a] * A.w[a] + B.w[b] * B.w[b] + C.w[c] * C.w[c]);
  *nodes += (long)A.m * B.m * C.m;
  return acc / (4 * M_PI);
}
static long prod_nodes(const rect* P, const rect* Q) {
  double d = gap(P, Q);
  return (long)qfor(0.5 * (P->a1 - P->a0), d) * qfor(0.5 * (P->b1 - P->b0), d) * qfor(0.5 * (Q->a1 - Q->a0), d) *
         qfor(0.5 * (Q->b1 - Q->b0), d);
}
int main(int argc, char** argv) {
  legendre_init();
  double tol = argc > 1 ? atof(argv[1]) : 1e-12;
  int N = argc > 2 ? atoi(argv[2]) : 200;
  for (int q = 1; q <= 16; ++q) {
    double rho = pow(tol, -1.0 / (2.0 * q));
    g_delta[q] = 0.5 * (rho + 1.0 / rho) - 1.0;
  }
  double gs[] = {1, 1.5, 2, 3, 4, 6, 8, 16, 32};
  for (int gi = 0; gi < 9; ++gi) {
    double worst = 0; long nt = 0, np = 0; int over = 0;
    for (int n = 0; n < N; ++n) {
      rect P, Q;
      P.axis = (int)(U() * 3); P.level = 0;
      double la = 0.2 + U(), asp = U() < 0.5 ? 1 : exp((U() * 2 - 1) * log(10.0)), lb = la * asp;
      P.a0 = -la / 2; P.a1 = la / 2; P.b0 = -lb / 2; P.b1 = lb / 2;
      int cls = (int)(U() * 3);
      Q.axis = cls < 2 ? P.axis : (P.axis + 1 + (int)(U() * 2)) % 3;
      double s = exp((U() * 2 - 1) * log(8.0));
      double lc = (0.2 + U()) * s, asp2 = U() < 0.5 ? 1 : exp((U() * 2 - 1) * log(10.0)), ld = lc * asp2;
      double dv[3] = {U() * 2 - 1, U() * 2 - 1, U() * 2 - 1};
      if (cls == 0) dv[P.axis] = 0;
      double nn = sqrt(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2]);
      for (int k = 0; k < 3; ++k) dv[k] /= nn;
      double dm = fmax(diam(&P), hypot(lc, ld)), lo = 0, hi = 200;
      for (int it = 0; it < 80; ++it) {
        double m = 0.5 * (lo + hi); int q0, q1; ip(Q.axis, &q0, &q1);
        Q.level = cls == 0 ? 0 : dv[Q.axis] * m;
        Q.a0 = dv[q0] * m - lc / 2; Q.a1 = dv[q0] * m + lc / 2; Q.b0 = dv[q1] * m - ld / 2; Q.b1 = dv[q1] * m + ld / 2;
        if (gap(&P, &Q) / dm < gs[gi]) lo = m; else hi = m;
      }
      double v = tent_rule(&P, &Q, &nt), tr = truth(&P, &Q);
      double e = fabs(v - tr) / tr;
      if (e > worst) worst = e;
      if (e > 1e-11) over++;
      np += prod_nodes(&P, &Q);
    }
    printf("g=%5.2f worst=%.2e over1e-11=%d mean_nodes tent=%.1f product=%.1f\n", gs[gi], worst, over, (double)nt / N,
           (double)np / N);
    fflush(stdout);
  }
  return 0;
}

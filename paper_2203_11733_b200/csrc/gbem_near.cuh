// gbem_near.cuh — near-field / singular pair integrals on the GPU.
//
// These classes (self, edge/corner-touching, and pairs closer than one
// diameters) are evaluated with the reference's own semi-analytic reductions,
// re-expressed for the GPU:
//   * coplanar: 16-corner closed form, one thread per pair
//     (uCoplanar/kCoplanar, proj/include/gbem/kernels.hpp:77-94);
//   * offset-parallel and orthogonal: the 1-D reduced integrands
//     (kernels.hpp:138-153, 175-214) integrated by the reference's Romberg rule
//     (quadrature.hpp:27-64) with its split-at-0 and t^4 endpoint substitution
//     (quadrature.hpp:70-113), ONE WARP PER PAIR: the odd samples of every
//     Romberg level are spread over the 32 lanes and reduced in a fixed tree
//     order, so the tableau and the stopping decision stay warp-uniform.
// Arithmetic follows the reference's evaluation order (this TU is compiled with
// -fmad=false), so results agree with the CPU reference to libm rounding.
#pragma once
#include "gbem_common.cuh"

namespace gbem_gpu {

constexpr int kRombMax = 20;  // hard cap on QuadratureConfig::maxLevels

// ---- closed-form helpers (kernels.hpp:48-62) ----
__device__ inline double d_log_u_plus_r(double u, double c2) {
  double r = sqrt(u * u + c2);
  if (u >= 0.0) {
    double arg = u + r;
    return arg > 0.0 ? log(arg) : -CUDART_INF;
  }
  if (c2 == 0.0) return -CUDART_INF;
  return log(c2) - log(r - u);
}

__device__ inline double d_mul_log(double pref, double u, double c2, double guard) {
  if (fabs(pref) <= guard) return 0.0;
  return pref * d_log_u_plus_r(u, c2);
}

// kCoplanar (kernels.hpp:77-84)
__device__ inline double d_k_coplanar(double u, double v, double guard) {
  double s = sqrt(u * u + v * v);
  double g1 = d_mul_log(0.5 * u * v * v, u, v * v, guard) - 0.75 * u * v * v +
              d_mul_log(u * u * v, v, u * u, guard) - 0.5 * u * u * s;
  double g2 = (u * u + v * v) * s / 6.0 + d_mul_log(0.5 * u * u * v, v, u * u, guard) -
              0.5 * u * u * s;
  return g1 - g2;
}

// uCorners (kernels.hpp:71-73): (+, xu-yd), (+, xd-yu), (-, xu-yu), (-, xd-yd)
struct Corners {
  double val[4];
  __device__ Corners(double xd, double xu, double yd, double yu) {
    val[0] = xu - yd;
    val[1] = xd - yu;
    val[2] = xu - yu;
    val[3] = xd - yd;
  }
  __device__ static double sign(int k) { return k < 2 ? 1.0 : -1.0; }
};

__device__ inline double dmax4(double a, double b, double c, double d) {
  double m = a;
  m = m < b ? b : m;
  m = m < c ? c : m;
  m = m < d ? d : m;
  return m;
}

// uCoplanar (kernels.hpp:86-94) on spans (sx,sy) of a and (tx,ty) of b.
__device__ inline double d_u_coplanar(double sx0, double sx1, double sy0, double sy1, double tx0,
                                      double tx1, double ty0, double ty1) {
  double scale = dmax4(sx1 - sx0, sy1 - sy0, tx1 - tx0, ty1 - ty0);
  double guard = 1e-14 * scale * scale * scale;
  Corners cu(sx0, sx1, tx0, tx1), cv(sy0, sy1, ty0, ty1);
  double acc = 0.0;
#pragma unroll 1
  for (int p = 0; p < 4; ++p)
#pragma unroll 1
    for (int q = 0; q < 4; ++q)
      acc += Corners::sign(p) * Corners::sign(q) * d_k_coplanar(cu.val[p], cv.val[q], guard);
  return acc / kFourPi;
}

// rectLess (kernels.hpp:257-263)
__device__ inline bool d_rect_less(const DPanel& a, const DPanel& b) {
  double ka[6] = {(double)a.axis, a.level, a.a0, a.a1, a.b0, a.b1};
  double kb[6] = {(double)b.axis, b.level, b.a0, b.a1, b.b0, b.b1};
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    if (ka[i] < kb[i]) return true;
    if (kb[i] < ka[i]) return false;
  }
  return false;
}

// ---- reduced 1-D integrands ----

// uParallelOffset integrand (kernels.hpp:143-151) with the Tent weight (101-103).
struct ParIntegrand {
  double val[4];
  double b2, t0, t3, plateau;
  __device__ double operator()(double v) const {
    double c2 = v * v + b2;
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      double u = val[k];
      double r = sqrt(u * u + c2);
      acc += Corners::sign(k) * (u * d_log_u_plus_r(u, c2) - r);
    }
    double m = v - t0;
    m = plateau < m ? plateau : m;
    m = (t3 - v) < m ? (t3 - v) : m;
    double w = 0.0 < m ? m : 0.0;
    return w * acc;
  }
};

// fx of uOrthogonal (kernels.hpp:183-199)
struct OrthFx {
  double val[4];
  double y2d, y2u, guard;
  __device__ double operator()(double x) const {
    double acc = 0.0;
    double x2 = x * x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      double cv = val[k];
      double u2 = cv * cv;
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        double sy = side == 0 ? 1.0 : -1.0;
        double y = side == 0 ? y2u : y2d;
        double c2 = x2 + y * y;
        double term = d_mul_log(0.5 * cv * y, cv, c2, guard) + d_mul_log(0.5 * u2, y, u2 + x2, guard);
        double r = sqrt(u2 + c2);
        double g3 = 0.5 * y * r + d_mul_log(0.5 * (x2 + u2), y, u2 + x2, guard);
        acc += Corners::sign(k) * sy * (term - g3);
      }
    }
    return acc;
  }
};

// fy of uOrthogonal (kernels.hpp:201-210)
struct OrthFy {
  double val[4];
  double x3d, x3u, guard;
  __device__ double operator()(double y) const {
    double acc = 0.0;
    double y2 = y * y;
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        double sx = side == 0 ? 1.0 : -1.0;
        double x = side == 0 ? x3u : x3d;
        double c2 = x * x + y2;
        acc += Corners::sign(k) * sx * d_mul_log(0.5 * val[k] * x, val[k], c2, guard);
      }
    return acc;
  }
};


// ---- fast forms of the reduced integrands for the fixed-rule near field:
// log(u + r) for u < 0 as log(c2 / (r - u)) (one log instead of the
// reference's log(c2) - log(r - u)), and the two mulLog terms of fx that share
// log(y + sqrt(y^2 + u^2 + x^2)) evaluate it once.  Guards as mulLog: a term
// whose prefactor is <= guard contributes 0 and its log is not evaluated.
__device__ __forceinline__ double d_lupr_fast(double u, double c2) {
  const double r = sqrt(u * u + c2);
  if (u >= 0.0) {
    const double arg = u + r;
    return arg > 0.0 ? log(arg) : -CUDART_INF;
  }
  return c2 == 0.0 ? -CUDART_INF : log(c2 / (r - u));
}

struct ParIntegrandFast {
  double val[4];
  double b2, t0, t3, plateau;
  __device__ double operator()(double v) const {
    const double c2 = v * v + b2;
    double acc = 0.0;
#pragma unroll 1
    for (int k = 0; k < 4; ++k) {
      const double u = val[k];
      const double r = sqrt(u * u + c2);
      const double lg = u >= 0.0 ? log(u + r) : log(c2 / (r - u));
      acc += Corners::sign(k) * (u * lg - r);
    }
    double m = v - t0;
    m = plateau < m ? plateau : m;
    m = (t3 - v) < m ? (t3 - v) : m;
    return (0.0 < m ? m : 0.0) * acc;
  }
};

struct OrthFxFast {
  double val[4];
  double y2d, y2u, guard;
  __device__ double operator()(double x) const {
    double acc = 0.0;
    const double x2 = x * x;
    // loops kept rolled: the log expansions appear once (instruction-cache footprint)
#pragma unroll 1
    for (int k = 0; k < 4; ++k) {
      const double cv = val[k];
      const double u2 = cv * cv;
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        const double y = side == 0 ? y2u : y2d;
        const double c2 = x2 + y * y;
        const double p1 = 0.5 * cv * y, p2 = 0.5 * u2, p3 = 0.5 * (x2 + u2);
        double term = 0.0;
        if (fabs(p1) > guard) term = p1 * d_lupr_fast(cv, c2);
        if (fabs(p2) > guard || fabs(p3) > guard) {
          const double l2 = d_lupr_fast(y, u2 + x2);
          if (fabs(p2) > guard) term += p2 * l2;
          term -= fabs(p3) > guard ? p3 * l2 : 0.0;
        }
        const double r = sqrt(u2 + c2);
        const double t = term - 0.5 * y * r;
        acc += (side == 0 ? Corners::sign(k) : -Corners::sign(k)) * t;
      }
    }
    return acc;
  }
};

struct OrthFyFast {
  double val[4];
  double x3d, x3u, guard;
  __device__ double operator()(double y) const {
    double acc = 0.0;
    const double y2 = y * y;
#pragma unroll 1
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        const double x = side == 0 ? x3u : x3d;
        const double p = 0.5 * val[k] * x;
        if (fabs(p) > guard) {
          const double t = p * d_lupr_fast(val[k], x * x + y2);
          acc += (side == 0 ? Corners::sign(k) : -Corners::sign(k)) * t;
        }
      }
    return acc;
  }
};

// t^4 endpoint substitution (quadrature.hpp:80-93): g(t) = 4 t^3 f(base +- t^4)
template <class F>
struct T4 {
  const F* f;
  double base;
  bool from_hi;
  __device__ double operator()(double t) const {
    if (t == 0.0) return 0.0;
    double t4 = t * t * t * t;
    double x = from_hi ? base - t4 : base + t4;
    return 4.0 * t * t * t * (*f)(x);
  }
};

struct WarpQuad {
  long evals = 0;
  bool converged = true;
  bool nonfinite = false;
};

// Warp sum with a fixed tree order and a broadcast from lane 0, so every lane
// holds bit-identical totals (keeps the Romberg decisions warp-uniform).
__device__ __forceinline__ double warp_sum_bcast(double x) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
  return __shfl_sync(0xffffffffu, x, 0);
}

// Evaluate f at one point on lane `src` and broadcast.
template <class F>
__device__ __forceinline__ double warp_point(const F& f, double x, int lane, int src) {
  double v = 0.0;
  if (lane == src) v = f(x);
  return __shfl_sync(0xffffffffu, v, src);
}

// romberg (quadrature.hpp:27-64), warp-cooperative.
template <class F>
__device__ double warp_romberg(const F& f, double a, double b, double rel_tol, int L, int lane,
                               WarpQuad& st) {
  if (a == b) return 0.0;
  double rowA[kRombMax + 1], rowB[kRombMax + 1];
  double* prev = rowA;
  double* cur = rowB;
  double fa = warp_point(f, a, lane, 0);
  double fb = warp_point(f, b, lane, 1 % 32);
  st.evals += 2;
  if (!isfinite(fa) || !isfinite(fb)) {
    st.nonfinite = true;
    return CUDART_NAN;
  }
  double h = b - a;
  prev[0] = 0.5 * h * (fa + fb);
  int hits = 0;
  for (int k = 1; k <= L; ++k) {
    h *= 0.5;
    long half = 1L << (k - 1);  // odd samples i = 2m+1, m < half
    double part = 0.0;
    bool bad = false;
    for (long m = lane; m < half; m += 32) {
      double s = f(a + (double)(2 * m + 1) * h);
      bad |= !isfinite(s);
      part += s;
    }
    st.evals += half;
    if (__any_sync(0xffffffffu, bad)) {
      st.nonfinite = true;
      return CUDART_NAN;
    }
    double tot = warp_sum_bcast(part);
    cur[0] = 0.5 * prev[0] + h * tot;
    double p4 = 1.0;
    for (int m = 1; m <= k; ++m) {
      p4 *= 4.0;
      cur[m] = cur[m - 1] + (cur[m - 1] - prev[m - 1]) / (p4 - 1.0);
    }
    if (k >= 4) {
      double diff = fabs(cur[k] - prev[k - 1]);
      double mag = fabs(cur[k]);
      mag = mag < 1e-300 ? 1e-300 : mag;
      hits = diff <= rel_tol * mag ? hits + 1 : 0;
      if (hits >= 2) return cur[k];
    }
    double* t = prev;
    prev = cur;
    cur = t;
  }
  st.converged = false;
  return prev[L];
}

// Romberg of the t^4-substituted integrand on a segment of length len whose
// singular endpoint is `base` (quadrature.hpp:80-93).
template <class F>
__device__ __noinline__ double warp_t4(const F& f, double base, double len, bool from_hi, double rel_tol,
                                       int L, int lane, WarpQuad& st) {
  T4<F> g{&f, base, from_hi};
  return warp_romberg(g, 0.0, sqrt(sqrt(len)), rel_tol, L, lane, st);
}

// integrateSegment (quadrature.hpp:70-94), recursion unrolled.
template <class F>
__device__ double warp_segment(const F& f, double a, double b, bool singA, bool singB,
                               double rel_tol, int L, int lane, WarpQuad& st) {
  if (a == b) return 0.0;
  if (singA && singB) {
    double m = 0.5 * (a + b);
    double left = m == a ? 0.0 : warp_t4(f, a, m - a, false, rel_tol, L, lane, st);
    if (st.nonfinite) return CUDART_NAN;
    double right = b == m ? 0.0 : warp_t4(f, b, b - m, true, rel_tol, L, lane, st);
    return left + right;
  }
  if (singA) return warp_t4(f, a, b - a, false, rel_tol, L, lane, st);
  if (singB) return warp_t4(f, b, b - a, true, rel_tol, L, lane, st);
  return warp_romberg(f, a, b, rel_tol, L, lane, st);
}

// integrateWithSplits (quadrature.hpp:98-113): split at 0 when interior,
// endpoint singularity probed with !isfinite(f(x)) (probes not counted).
template <class F>
__device__ double warp_with_splits(const F& f, double a, double b, double rel_tol, int L, int lane,
                                   WarpQuad& st) {
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
    bool sa = !isfinite(warp_point(f, pts[i], lane, 0));
    bool sb = !isfinite(warp_point(f, pts[i + 1], lane, 0));
    total += warp_segment(f, pts[i], pts[i + 1], sa, sb, rel_tol, L, lane, st);
    if (st.nonfinite) return CUDART_NAN;
  }
  return total;
}

// std::sort of <= 5 doubles (tentSegments' sort, kernels.hpp:119)
__device__ inline void sort5(double* p, int n) {
  for (int i = 1; i < n; ++i) {
    double x = p[i];
    int j = i - 1;
    while (j >= 0 && x < p[j]) {
      p[j + 1] = p[j];
      --j;
    }
    p[j + 1] = x;
  }
}

// uParallelOffset (kernels.hpp:138-153) for canonical (a, b), b = a.level - b.level.
__device__ inline double warp_u_parallel(const DPanel& A, const DPanel& B, double rel_tol, int L,
                                         int lane, WarpQuad& st) {
  double off = A.level - B.level;
  ParIntegrand f;
  Corners c(A.a0, A.a1, B.a0, B.a1);
  for (int k = 0; k < 4; ++k) f.val[k] = c.val[k];
  f.b2 = off * off;
  // tentSegments (kernels.hpp:112-125) on (sy, ty) = (A.b, B.b)
  double xd = A.b0, xu = A.b1, yd = B.b0, yu = B.b1;
  double t0 = xd - yu, t3 = xu - yd;
  double da = xd - yd, db = xu - yu;
  double k1 = db < da ? db : da;
  double k2 = da < db ? db : da;
  f.t0 = t0;
  f.t3 = t3;
  f.plateau = (yu - yd) < (xu - xd) ? (yu - yd) : (xu - xd);
  double pts[5] = {t0, k1, k2, t3, 0.0};
  int n = 4;
  if (t0 < 0.0 && 0.0 < t3) n = 5;
  sort5(pts, n);
  double cuts[5];
  int count = 0;
  for (int i = 0; i < n; ++i)
    if (count == 0 || pts[i] > cuts[count - 1]) cuts[count++] = pts[i];
  double total = 0.0;
  for (int i = 0; i + 1 < count; ++i) {
    total += warp_romberg(f, cuts[i], cuts[i + 1], rel_tol, L, lane, st);
    if (st.nonfinite) return CUDART_NAN;
  }
  return total / kFourPi;
}

// orthFrame + uOrthogonal (kernels.hpp:175-214, 245-255) for canonical (a, b).
__device__ inline double warp_u_orthogonal(const DPanel& A, const DPanel& B, double rel_tol, int L,
                                           int lane, WarpQuad& st) {
  int shared = 3 - A.axis - B.axis;
  double s1lo, s1hi, t1lo, t1hi, i3lo, i3hi, j2lo, j2hi;
  panel_extent(A, shared, s1lo, s1hi);
  panel_extent(B, shared, t1lo, t1hi);
  panel_extent(A, B.axis, i3lo, i3hi);
  panel_extent(B, A.axis, j2lo, j2hi);
  double s3lo = i3lo - B.level, s3hi = i3hi - B.level;
  double t2lo = j2lo - A.level, t2hi = j2hi - A.level;
  Corners c(s1lo, s1hi, t1lo, t1hi);
  double scale = dmax4(s1hi - s1lo, t1hi - t1lo, s3hi - s3lo, t2hi - t2lo);
  scale = scale < 1e-30 ? 1e-30 : scale;
  double guard = 1e-14 * scale;
  OrthFx fx;
  OrthFy fy;
  for (int k = 0; k < 4; ++k) {
    fx.val[k] = c.val[k];
    fy.val[k] = c.val[k];
  }
  fx.y2d = t2lo;
  fx.y2u = t2hi;
  fx.guard = guard;
  fy.x3d = s3lo;
  fy.x3u = s3hi;
  fy.guard = guard;
  double tx = warp_with_splits(fx, s3lo, s3hi, rel_tol, L, lane, st);
  if (st.nonfinite) return CUDART_NAN;
  double ty = warp_with_splits(fy, t2lo, t2hi, rel_tol, L, lane, st);
  if (st.nonfinite) return CUDART_NAN;
  return (tx + ty) / kFourPi;
}

// ---- double layer (kernels.hpp:157-169, 218-237, 295-315), warp-cooperative
// Romberg as the reference: test panel I, source panel J; the caller applies
// the source normal sign.

// qParallelOffset integrand (kernels.hpp:162-167): w(v) * sum_k s_k sqrt(u_k^2 + c2) / c2
struct QParIntegrand {
  double val[4];
  double b2, t0, t3, plateau;
  __device__ double operator()(double v) const {
    const double c2 = v * v + b2;
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) acc += Corners::sign(k) * sqrt(val[k] * val[k] + c2) / c2;
    double m = v - t0;
    m = plateau < m ? plateau : m;
    m = (t3 - v) < m ? (t3 - v) : m;
    const double w = 0.0 < m ? m : 0.0;
    return w * acc;
  }
};

// fy of qOrthogonal (kernels.hpp:224-235)
struct QOrthFy {
  double val[4];
  double x3d, x3u, guard;
  __device__ double operator()(double y) const {
    double acc = 0.0;
    const double y2 = y * y;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const double s3s = side == 0 ? 1.0 : -1.0;
      const double x3 = side == 0 ? x3d : x3u;
      const double c2 = y2 + x3 * x3;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double r = sqrt(val[k] * val[k] + c2);
        acc += s3s * Corners::sign(k) * (d_mul_log(val[k], val[k], c2, guard) - r);
      }
    }
    return acc;
  }
};

// qParallelOffset for test I over source J, b = I.level - J.level != 0
__device__ inline double warp_q_parallel(const DPanel& I, const DPanel& J, double rel_tol, int L, int lane,
                                         WarpQuad& st) {
  const double off = I.level - J.level;
  QParIntegrand f;
  Corners c(I.a0, I.a1, J.a0, J.a1);
  for (int k = 0; k < 4; ++k) f.val[k] = c.val[k];
  f.b2 = off * off;
  const double xd = I.b0, xu = I.b1, yd = J.b0, yu = J.b1;
  const double t0 = xd - yu, t3 = xu - yd;
  const double da = xd - yd, db = xu - yu;
  f.t0 = t0;
  f.t3 = t3;
  f.plateau = (yu - yd) < (xu - xd) ? (yu - yd) : (xu - xd);
  double pts[5] = {t0, db < da ? db : da, da < db ? db : da, t3, 0.0};
  int n = (t0 < 0.0 && 0.0 < t3) ? 5 : 4;
  sort5(pts, n);
  double cuts[5];
  int count = 0;
  for (int i = 0; i < n; ++i)
    if (count == 0 || pts[i] > cuts[count - 1]) cuts[count++] = pts[i];
  double total = 0.0;
  for (int i = 0; i + 1 < count; ++i) {
    total += warp_romberg(f, cuts[i], cuts[i + 1], rel_tol, L, lane, st);
    if (st.nonfinite) return CUDART_NAN;
  }
  return off * total / kFourPi;
}

// orthFrame(I, J) + qOrthogonal (kernels.hpp:218-237, 245-255)
__device__ inline double warp_q_orthogonal(const DPanel& I, const DPanel& J, double rel_tol, int L, int lane,
                                           WarpQuad& st) {
  const int shared = 3 - I.axis - J.axis;
  double s1lo, s1hi, t1lo, t1hi, i3lo, i3hi, j2lo, j2hi;
  panel_extent(I, shared, s1lo, s1hi);
  panel_extent(J, shared, t1lo, t1hi);
  panel_extent(I, J.axis, i3lo, i3hi);
  panel_extent(J, I.axis, j2lo, j2hi);
  const double s3lo = i3lo - J.level, s3hi = i3hi - J.level;
  const double t2lo = j2lo - I.level, t2hi = j2hi - I.level;
  Corners c(s1lo, s1hi, t1lo, t1hi);
  double scale = dmax4(s1hi - s1lo, t1hi - t1lo, s3hi - s3lo, t2hi - t2lo);
  scale = scale < 1e-30 ? 1e-30 : scale;
  QOrthFy fy;
  for (int k = 0; k < 4; ++k) fy.val[k] = c.val[k];
  fy.x3d = s3lo;
  fy.x3u = s3hi;
  fy.guard = 1e-14 * scale;
  const double ty = warp_with_splits(fy, t2lo, t2hi, rel_tol, L, lane, st);
  if (st.nonfinite) return CUDART_NAN;
  return ty / kFourPi;
}

// ---------------------------------------------------------------------------
// Fixed-cost near field: the same reduced integrands, each reference segment
// split at its midpoint and both halves integrated with x = end -+ t^2 grading
// toward their outer ends and an n-point Gauss-Legendre rule in t (nodes never
// touch an endpoint, so endpoint singularities need no probing).  Calibrated in
// tools/near_gl_experiment.c against the tight-tolerance reference algorithm:
// touching pairs <= 6e-13 with n = 20; gap/diam >= 0.1: n = 20, >= 0.02: n = 24,
// >= 0.005: n = 32, >= 1e-3: n = 48 (<= 1e-11 worst).  One thread per pair.

constexpr int kNearBands = 4;
__host__ __device__ constexpr int near_nodes(int band) {
  return band == 0 ? 20 : band == 1 ? 24 : band == 2 ? 32 : 48;
}

// A pair's nodes are shared by a team of kNearTeam consecutive lanes: lane tl
// of the team evaluates nodes tl, tl + kNearTeam, ...; the functions below
// return that lane's partial sum (linear in the nodes) and the kernel sums
// the team's partials (k_near_gl).
constexpr int kNearTeam = 4;

template <class F>
__device__ __noinline__ double gl_graded(const F& f, double a, double b, int band, const double (*nx)[48],
                            const double (*nw)[48], bool& bad, int tl) {
  if (a == b) return 0.0;
  const int n = near_nodes(band);
  const double m = 0.5 * (a + b);
  double total = 0.0;
#pragma unroll 1
  for (int side = 0; side < 2; ++side) {
    const double base = side ? b : a;
    const double len = side ? b - m : m - a;
    const double h = 0.5 * sqrt(len);
    double part = 0.0;
#pragma unroll 1
    for (int i = tl; i < n; i += kNearTeam) {
      const double t = fma(h, nx[band][i], h);
      const double x = side ? base - t * t : base + t * t;
      const double v = f(x);
      bad |= !isfinite(v);
      part = fma(nw[band][i] * t, v, part);
    }
    total += 2.0 * h * part;
  }
  return total;
}

// uParallelOffset (kernels.hpp:138-153) with the graded Gauss rule.
__device__ inline double gl_u_parallel(const DPanel& A, const DPanel& B, int band, const double (*nx)[48],
                                       const double (*nw)[48], bool& bad, int tl) {
  double off = A.level - B.level;
  ParIntegrandFast f;
  Corners c(A.a0, A.a1, B.a0, B.a1);
  for (int k = 0; k < 4; ++k) f.val[k] = c.val[k];
  f.b2 = off * off;
  double xd = A.b0, xu = A.b1, yd = B.b0, yu = B.b1;
  double t0 = xd - yu, t3 = xu - yd;
  double da = xd - yd, db = xu - yu;
  f.t0 = t0;
  f.t3 = t3;
  f.plateau = (yu - yd) < (xu - xd) ? (yu - yd) : (xu - xd);
  double pts[5] = {t0, db < da ? db : da, da < db ? db : da, t3, 0.0};
  int n = (t0 < 0.0 && 0.0 < t3) ? 5 : 4;
  sort5(pts, n);
  double cuts[5];
  int count = 0;
  for (int i = 0; i < n; ++i)
    if (count == 0 || pts[i] > cuts[count - 1]) cuts[count++] = pts[i];
  double total = 0.0;
  for (int i = 0; i + 1 < count; ++i) total += gl_graded(f, cuts[i], cuts[i + 1], band, nx, nw, bad, tl);
  return total / kFourPi;
}

template <class F>
__device__ double gl_split0(const F& f, double a, double b, int band, const double (*nx)[48],
                            const double (*nw)[48], bool& bad, int tl) {
  if (a < 0.0 && 0.0 < b)
    return gl_graded(f, a, 0.0, band, nx, nw, bad, tl) + gl_graded(f, 0.0, b, band, nx, nw, bad, tl);
  return gl_graded(f, a, b, band, nx, nw, bad, tl);
}

// orthFrame + uOrthogonal (kernels.hpp:175-214, 245-255) with the graded Gauss rule.
__device__ inline double gl_u_orthogonal(const DPanel& A, const DPanel& B, int band, const double (*nx)[48],
                                         const double (*nw)[48], bool& bad, int tl) {
  int shared = 3 - A.axis - B.axis;
  double s1lo, s1hi, t1lo, t1hi, i3lo, i3hi, j2lo, j2hi;
  panel_extent(A, shared, s1lo, s1hi);
  panel_extent(B, shared, t1lo, t1hi);
  panel_extent(A, B.axis, i3lo, i3hi);
  panel_extent(B, A.axis, j2lo, j2hi);
  double s3lo = i3lo - B.level, s3hi = i3hi - B.level;
  double t2lo = j2lo - A.level, t2hi = j2hi - A.level;
  Corners c(s1lo, s1hi, t1lo, t1hi);
  double scale = dmax4(s1hi - s1lo, t1hi - t1lo, s3hi - s3lo, t2hi - t2lo);
  scale = scale < 1e-30 ? 1e-30 : scale;
  OrthFxFast fx;
  OrthFyFast fy;
  for (int k = 0; k < 4; ++k) {
    fx.val[k] = c.val[k];
    fy.val[k] = c.val[k];
  }
  fx.y2d = t2lo;
  fx.y2u = t2hi;
  fx.guard = 1e-14 * scale;
  fy.x3d = s3lo;
  fy.x3u = s3hi;
  fy.guard = fx.guard;
  double tx = gl_split0(fx, s3lo, s3hi, band, nx, nw, bad, tl);
  double ty = gl_split0(fy, t2lo, t2hi, band, nx, nw, bad, tl);
  return (tx + ty) / kFourPi;
}

}  // namespace gbem_gpu

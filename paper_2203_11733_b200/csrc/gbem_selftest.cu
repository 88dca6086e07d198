// gbem_selftest.cu — the randomised kernel audit of the reference
// (run_selftest, proj/include/gbem/selftest.hpp:184-245) on the GPU.
//
// Ten geometric case classes (the generators of selftest.hpp:60-161, drawn
// from a counter-based splitmix64 stream instead of std::mt19937_64, whose
// real distributions are library-defined), each checked against the
// brute-force oracle of oracle.hpp:44-205 -- recursive dyadic subdivision
// toward the closest-approach region, the exact half-scale relation for
// identical rectangles, presplit at the other panel's extents and a 6^4
// tensor Gauss rule on well-separated leaves -- evaluated on the device:
//   semi-analytic U = the production pair evaluators (gbem_u_pair_integrals:
//                     far-field difference-set Gauss, graded near field,
//                     coplanar closed form, Romberg near contact);
//   semi-analytic Q = the double-layer kernel (warp_q_parallel / _orthogonal);
//   oracle          = one warp per pair walking an explicit DFS stack in shared
//                     memory, the 1,296 Gauss nodes of a leaf spread over the
//                     lanes; touching classes use the Aitken extrapolation of
//                     depths 3, 4, 5 (selftest.hpp:33-52), disjoint ones depth 6.
// Per class: worst relErr = |semi - oracle| / max(|oracle|, 1e-9) against the
// reference's tolerances (1e-6 disjoint, 1e-3 touching, 1e-12 for the
// vanishing coplanar double layer).
#include <cstring>
#include <string>
#include <vector>

#include "gbem_ctx.cuh"
#include "gbem_near.cuh"

using namespace gbem_gpu;

namespace {

// ------------------------------------------------------------ generators

struct Rng {
  unsigned long long s;
  __device__ unsigned long long next() {  // splitmix64
    unsigned long long z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  __device__ double uni(double lo, double hi) { return lo + (hi - lo) * ((next() >> 11) * (1.0 / 9007199254740992.0)); }
  __device__ double gauss() {  // Box-Muller
    const double u1 = ((next() >> 11) + 1) * (1.0 / 9007199254740993.0), u2 = uni(0.0, 1.0);
    return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
  __device__ int pick(int n) { return (int)(next() % (unsigned long long)n); }
  __device__ bool coin() { return (next() & 1ull) != 0; }
};

struct GRect {
  DPanel g;
  int ns;
};

__device__ void rspan(Rng& r, double& lo, double& hi) {
  lo = r.uni(-2.0, 2.0);
  hi = lo + r.uni(0.3, 2.0);
}
__device__ GRect coplanar_base(Rng& r, int axis, double lv) {
  GRect o;
  o.g.axis = axis;
  o.g.pad = 0;
  o.g.level = lv;
  rspan(r, o.g.a0, o.g.a1);
  rspan(r, o.g.b0, o.g.b1);
  o.ns = r.coin() ? 1 : -1;
  return o;
}

// selftest.hpp:80-159 (cases: 0 copDisjoint, 1 copAdjacent, 2 copIdentical,
// 3 parOffset, 4 orthDisjoint, 5 orthAdjacent)
__device__ void gen_pair(int gen, Rng& r, GRect& a, GRect& b) {
  if (gen == 0) {
    const int axis = r.pick(3);
    const double lv = r.gauss();
    for (;;) {
      a = coplanar_base(r, axis, lv);
      b = coplanar_base(r, axis, lv);
      const double g0 = fmax(b.g.a0 - a.g.a1, a.g.a0 - b.g.a1), g1 = fmax(b.g.b0 - a.g.b1, a.g.b0 - b.g.b1);
      if (fmax(g0, g1) > 0.05) return;
    }
  } else if (gen == 1) {
    const int axis = r.pick(3);
    const double lv = r.gauss();
    a = coplanar_base(r, axis, lv);
    b = coplanar_base(r, axis, lv);
    const bool alongA = r.coin(), hiSide = r.coin();
    const double w = r.uni(0.3, 2.0);
    const double rlo = alongA ? a.g.a0 : a.g.b0, rhi = alongA ? a.g.a1 : a.g.b1;
    const double lo = hiSide ? rhi : rlo - w, hi = hiSide ? rhi + w : rlo;
    if (alongA) {
      b.g.a0 = lo;
      b.g.a1 = hi;
    } else {
      b.g.b0 = lo;
      b.g.b1 = hi;
    }
  } else if (gen == 2) {
    const int axis = r.pick(3);
    a = coplanar_base(r, axis, r.gauss());
    b = a;
  } else if (gen == 3) {
    const int axis = r.pick(3);
    const double lv = r.gauss();
    const double off = r.uni(0.3, 2.0) * (r.coin() ? 1.0 : -1.0);
    a = coplanar_base(r, axis, lv);
    b = coplanar_base(r, axis, lv + off);
  } else if (gen == 4) {
    for (;;) {
      const int ax1 = r.pick(3), ax2 = (ax1 + 1 + r.pick(2)) % 3;
      a = coplanar_base(r, ax1, r.gauss());
      b = coplanar_base(r, ax2, r.gauss());
      if (panel_gap(a.g, b.g) > 0.05) return;
    }
  } else {
    const int ax1 = r.pick(3), ax2 = (ax1 + 1 + r.pick(2)) % 3, shared = 3 - ax1 - ax2;
    const double lv1 = r.gauss(), lv2 = r.gauss();
    const double w1 = r.uni(0.3, 2.0), w2 = r.uni(0.3, 2.0);
    double e1lo, e1hi, e2lo, e2hi;
    if (r.coin()) { e1lo = lv2; e1hi = lv2 + w1; } else { e1lo = lv2 - w1; e1hi = lv2; }
    if (r.coin()) { e2lo = lv1; e2hi = lv1 + w2; } else { e2lo = lv1 - w2; e2hi = lv1; }
    auto mk = [&](int axis, double lv, double elo, double ehi) {
      GRect o;
      o.g.axis = axis;
      o.g.pad = 0;
      o.g.level = lv;
      o.ns = r.coin() ? 1 : -1;
      double slo, shi;
      rspan(r, slo, shi);
      if (ip0(axis) == shared) {
        o.g.a0 = slo; o.g.a1 = shi; o.g.b0 = elo; o.g.b1 = ehi;
      } else {
        o.g.a0 = elo; o.g.a1 = ehi; o.g.b0 = slo; o.g.b1 = shi;
      }
      return o;
    };
    a = mk(ax1, lv1, e1lo, e1hi);
    b = mk(ax2, lv2, e2lo, e2hi);
  }
}

// pair t of a class -> panels t (test) and npairs + t (source) of the context's
// panel array, and the source normal sign
__global__ void k_st_gen(int gen, unsigned long long seed, int npairs, DPanel* P, int* nsign) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= npairs) return;
  Rng r{seed ^ ((unsigned long long)(gen + 1) << 52) ^ ((unsigned long long)t * 0xD1B54A32D192ED03ull)};
  GRect a, b;
  gen_pair(gen, r, a, b);
  P[t] = a.g;
  P[npairs + t] = b.g;
  nsign[t] = b.ns;
}

// ------------------------------------------------------------ semi-analytic Q

// q_pair_integral (kernels.hpp:295-315): one warp per pair
__global__ void __launch_bounds__(128) k_st_q(const DPanel* __restrict__ P, const int* __restrict__ nsign, int npairs,
                                              double rel_tol, int max_levels, double* out) {
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (t >= npairs) return;
  const DPanel I = P[t], J = P[npairs + t];
  WarpQuad st;
  double q = 0.0;
  if (I.axis != J.axis)
    q = warp_q_orthogonal(I, J, rel_tol, max_levels, lane, st);
  else if (I.level != J.level)
    q = warp_q_parallel(I, J, rel_tol, max_levels, lane, st);
  if (lane == 0) out[t] = (double)nsign[t] * q;
}

// ------------------------------------------------------------ brute-force oracle

__constant__ double c_g6x[6] = {-0.9324695142031520278123016, -0.6612093864662645136613996,
                                -0.2386191860831969086305017, 0.2386191860831969086305017,
                                0.6612093864662645136613996,  0.9324695142031520278123016};
__constant__ double c_g6w[6] = {0.1713244923791703450402961, 0.3607615730481386075698335,
                                0.4679139345726910473898703, 0.4679139345726910473898703,
                                0.3607615730481386075698335, 0.1713244923791703450402961};

struct StackEntry {
  DPanel r1, r2;
  double wt;
  int depth, pad;
};
constexpr int kStack = 192;         // 81 presplit pairs + 6 levels x 16 children, with room
constexpr int kOracleWarps = 2;     // warps per CTA (each with its own stack)

__device__ __forceinline__ bool same_geometry(const DPanel& a, const DPanel& b) {
  return a.axis == b.axis && a.level == b.level && a.a0 == b.a0 && a.a1 == b.a1 && a.b0 == b.b0 && a.b1 == b.b1;
}
__device__ __forceinline__ double diam(const DPanel& r) { return hypot(r.a1 - r.a0, r.b1 - r.b0); }
__device__ __forceinline__ DPanel child(const DPanel& r, int k) {  // split4 (oracle.hpp:21-35)
  const double ma = 0.5 * (r.a0 + r.a1), mb = 0.5 * (r.b0 + r.b1);
  DPanel c = r;
  if (k & 1) c.a0 = ma; else c.a1 = ma;
  if (k & 2) c.b0 = mb; else c.b1 = mb;
  return c;
}

// gaussPair (oracle.hpp:44-81) of U* (single layer) or Q* (double layer, source
// normal along r2.axis with sign ns), this lane's share of the 1,296 nodes
__device__ double gauss_pair_lane(const DPanel& r1, const DPanel& r2, bool dbl, int ns, int lane) {
  const int i0 = ip0(r1.axis), i1 = ip1(r1.axis), j0 = ip0(r2.axis), j1 = ip1(r2.axis);
  const double ca = 0.5 * (r1.a0 + r1.a1), ha = 0.5 * (r1.a1 - r1.a0), cb = 0.5 * (r1.b0 + r1.b1),
               hb = 0.5 * (r1.b1 - r1.b0);
  const double cc = 0.5 * (r2.a0 + r2.a1), hc = 0.5 * (r2.a1 - r2.a0), cd = 0.5 * (r2.b0 + r2.b1),
               hd = 0.5 * (r2.b1 - r2.b0);
  double acc = 0.0;
  for (int idx = lane; idx < 1296; idx += 32) {
    const int i = idx / 216, j = (idx / 36) % 6, k = (idx / 6) % 6, l = idx % 6;
    double p[3], q[3];
    p[r1.axis] = r1.level;
    p[i0] = fma(ha, c_g6x[i], ca);
    p[i1] = fma(hb, c_g6x[j], cb);
    q[r2.axis] = r2.level;
    q[j0] = fma(hc, c_g6x[k], cc);
    q[j1] = fma(hd, c_g6x[l], cd);
    const double w = (ha * c_g6w[i]) * (hb * c_g6w[j]) * (hc * c_g6w[k]) * (hd * c_g6w[l]);
    const double dx = p[0] - q[0], dy = p[1] - q[1], dz = p[2] - q[2];
    const double r2s = dx * dx + dy * dy + dz * dz;
    double kern;
    if (!dbl) {
      kern = 1.0 / (kFourPi * sqrt(r2s));
    } else {
      const double dn = (p[r2.axis] - q[r2.axis]) * (double)ns;
      kern = dn / (kFourPi * r2s * sqrt(r2s));
    }
    acc = fma(w, kern, acc);
  }
  return acc;
}

// cut [lo, hi] at the interior points c0, c1 (oracle.hpp:134-143)
__device__ int cut_span(double lo, double hi, double c0, double c1, double* pts) {
  int n = 0;
  pts[n++] = lo;
  pts[n++] = hi;
  if (c0 > lo && c0 < hi) pts[n++] = c0;
  if (c1 > lo && c1 < hi && c1 != c0) pts[n++] = c1;
  for (int i = 1; i < n; ++i) {  // sort
    const double x = pts[i];
    int j = i - 1;
    while (j >= 0 && x < pts[j]) {
      pts[j + 1] = pts[j];
      --j;
    }
    pts[j + 1] = x;
  }
  return n;
}

// oracle_pair_integral (oracle.hpp:191-205), one warp per pair; `dbl` selects
// recQ (oracle.hpp:105-131) over recU (oracle.hpp:90-103).
__global__ void __launch_bounds__(32 * kOracleWarps)
    k_st_oracle(const DPanel* __restrict__ P, const int* __restrict__ nsign, int npairs, int dbl, int depth,
                double* out) {
  __shared__ StackEntry stk[kOracleWarps][kStack];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * kOracleWarps + w;
  if (t >= npairs) return;
  StackEntry* S = stk[w];
  const DPanel Ii = P[t], Ij = P[npairs + t];
  const int ns = nsign[t];
  int top = 0;
  double acc = 0.0;
  const bool coplanar = Ii.axis == Ij.axis && Ii.level == Ij.level;
  if (dbl && coplanar) {
    if (lane == 0) out[t] = 0.0;
    return;
  }
  if (lane == 0) {
    if (!dbl && same_geometry(Ii, Ij)) {
      S[top++] = StackEntry{Ii, Ij, 1.0, depth, 0};
    } else {
      // presplit(Ii, Ij) x presplit(Ij, Ii)
      double pa1[4], pb1[4], pa2[4], pb2[4];
      double lo, hi, lo2, hi2;
      panel_extent(Ij, ip0(Ii.axis), lo, hi);
      panel_extent(Ij, ip1(Ii.axis), lo2, hi2);
      const int na1 = cut_span(Ii.a0, Ii.a1, lo, hi, pa1), nb1 = cut_span(Ii.b0, Ii.b1, lo2, hi2, pb1);
      panel_extent(Ii, ip0(Ij.axis), lo, hi);
      panel_extent(Ii, ip1(Ij.axis), lo2, hi2);
      const int na2 = cut_span(Ij.a0, Ij.a1, lo, hi, pa2), nb2 = cut_span(Ij.b0, Ij.b1, lo2, hi2, pb2);
      for (int x = 0; x + 1 < na1; ++x)
        for (int y = 0; y + 1 < nb1; ++y)
          for (int u = 0; u + 1 < na2; ++u)
            for (int v = 0; v + 1 < nb2; ++v) {
              DPanel p1 = Ii, p2 = Ij;
              p1.a0 = pa1[x]; p1.a1 = pa1[x + 1]; p1.b0 = pb1[y]; p1.b1 = pb1[y + 1];
              p2.a0 = pa2[u]; p2.a1 = pa2[u + 1]; p2.b0 = pb2[v]; p2.b1 = pb2[v + 1];
              S[top++] = StackEntry{p1, p2, 1.0, depth, 0};
            }
    }
  }
  top = __shfl_sync(0xffffffffu, top, 0);
  __syncwarp();
  while (top > 0) {
    const StackEntry e = S[top - 1];
    __syncwarp();
    --top;
    bool leaf = false;
    int push = 0;  // 1: identical half-scale, 2: both split, 3: larger split
    if (!dbl && same_geometry(e.r1, e.r2)) {
      push = 1;
    } else if (dbl && e.r1.axis == e.r2.axis && e.r1.level == e.r2.level) {
      continue;  // coplanar double layer vanishes
    } else {
      const double d = panel_gap(e.r1, e.r2), dm = fmax(diam(e.r1), diam(e.r2));
      if (d >= dm || e.depth <= 0)
        leaf = true;
      else
        push = d == 0.0 ? 2 : 3;
    }
    if (leaf) {
      acc = fma(e.wt, gauss_pair_lane(e.r1, e.r2, dbl, ns, lane), acc);
      continue;
    }
    if (lane == 0) {
      if (push == 1) {
        // U = 2 * (4a + 4b + 4c) over the translation classes of the 12 cross pairs
        const DPanel k0 = child(e.r1, 0);
        const double wa = 0.5 * (e.r1.a1 - e.r1.a0), hb = 0.5 * (e.r1.b1 - e.r1.b0);
        DPanel s1 = k0, s2 = k0, s3 = k0;
        s1.a0 += wa; s1.a1 += wa;
        s2.b0 += hb; s2.b1 += hb;
        s3.a0 += wa; s3.a1 += wa; s3.b0 += hb; s3.b1 += hb;
        S[top++] = StackEntry{k0, s1, 8.0 * e.wt, e.depth - 1, 0};
        S[top++] = StackEntry{k0, s2, 8.0 * e.wt, e.depth - 1, 0};
        S[top++] = StackEntry{k0, s3, 8.0 * e.wt, e.depth - 1, 0};
      } else if (push == 2) {
        for (int a = 0; a < 4; ++a)
          for (int b = 0; b < 4; ++b) S[top++] = StackEntry{child(e.r1, a), child(e.r2, b), e.wt, e.depth - 1, 0};
      } else {
        const bool first = diam(e.r1) >= diam(e.r2);
        for (int a = 0; a < 4; ++a)
          S[top++] = first ? StackEntry{child(e.r1, a), e.r2, e.wt, e.depth - 1, 0}
                           : StackEntry{e.r1, child(e.r2, a), e.wt, e.depth - 1, 0};
      }
    }
    top = __shfl_sync(0xffffffffu, top, 0);
    __syncwarp();
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) out[t] = acc;
}

// selftest.hpp:33-39
__device__ double aitken(double v0, double v1, double v2) {
  const double d1 = v1 - v0, d2 = v2 - v1, den = d2 - d1;
  if (fabs(den) < 1e-14 * fmax(fabs(v2), 1e-300)) return v2;
  return v2 - d2 * d2 / den;
}

// worst error of the class: mode 0 relErr vs o2 (disjoint), 1 relErr vs
// Aitken(o0, o1, o2) (touching), 2 |semi| + |o2| (vanishing coplanar Q)
__global__ void k_st_worst(const double* semi, const double* o0, const double* o1, const double* o2, int npairs,
                           int mode, unsigned long long* worst, double* err, double* ref_out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  double e = 0.0;
  if (t < npairs) {
    double ref = o2[t];
    if (mode == 2) {
      e = fabs(semi[t]) + fabs(o2[t]);
    } else {
      ref = mode == 1 ? aitken(o0[t], o1[t], o2[t]) : o2[t];
      e = fabs(semi[t] - ref) / fmax(fabs(ref), 1e-9);  // relErr (selftest.hpp:57-59)
    }
    if (!(e == e)) e = 1e300;  // NaN fails the class
    err[t] = e;
    ref_out[t] = ref;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) e = fmax(e, __shfl_xor_sync(0xffffffffu, e, off));
  if ((threadIdx.x & 31) == 0) atomicMax(worst, (unsigned long long)__double_as_longlong(e));
}

struct CaseDef {
  const char* name;
  int gen;
  int dbl;
  int mode;  // 0 disjoint (depth 6), 1 touching (Aitken 3/4/5), 2 Q coplanar zero (depth 3)
  double tol;
};
// selftest.hpp:212-233
const CaseDef kCases[10] = {
    {"U coplanar disjoint", 0, 0, 0, 1e-6}, {"U coplanar adjacent", 1, 0, 1, 1e-3},
    {"U coplanar identical", 2, 0, 1, 1e-3}, {"U parallel offset", 3, 0, 0, 1e-6},
    {"U orthogonal disjoint", 4, 0, 0, 1e-6}, {"U orthogonal adjacent", 5, 0, 1, 1e-3},
    {"Q coplanar zero", 1, 1, 2, 1e-12},     {"Q parallel offset", 3, 1, 0, 1e-6},
    {"Q orthogonal disjoint", 4, 1, 0, 1e-6}, {"Q orthogonal adjacent", 5, 1, 1, 1e-3},
};

}  // namespace

int gbem_internal_oracle_pairs(gbem_ctx* ctx, const gbem_panels* I, const gbem_panels* J, const int32_t* nsign,
                               int64_t npairs, int32_t dbl, int32_t depth, double* out) {
  if (npairs < 0 || npairs > (1 << 22)) return ctx->fail(GBEM_EINVAL, "npairs must be in [0, 2^22]");
  if (depth < 0 || depth > 6) return ctx->fail(GBEM_EINVAL, "oracle depth must be in [0, 6]");
  if (!I || !J || !out) return ctx->fail(GBEM_EINVAL, "null argument");
  if (npairs == 0) return GBEM_OK;
  // I then J as one 2 npairs panel list in the context's panel array
  const size_t n = (size_t)npairs;
  std::vector<uint8_t> ax(2 * n);
  std::vector<double> lv(2 * n), a0(2 * n), a1(2 * n), b0(2 * n), b1(2 * n);
  const gbem_panels* src[2] = {I, J};
  for (int s = 0; s < 2; ++s)
    for (size_t k = 0; k < n; ++k) {
      ax[s * n + k] = src[s]->axis[k];
      lv[s * n + k] = src[s]->level[k];
      a0[s * n + k] = src[s]->a_lo[k];
      a1[s * n + k] = src[s]->a_hi[k];
      b0[s * n + k] = src[s]->b_lo[k];
      b1[s * n + k] = src[s]->b_hi[k];
    }
  gbem_panels all{ax.data(), lv.data(), a0.data(), a1.data(), b0.data(), b1.data()};
  int rc = gbem_internal_upload_panels(ctx, &all, 2 * npairs, false);
  if (rc) return rc;
  std::vector<int> ns(n, 1);
  if (nsign)
    for (size_t k = 0; k < n; ++k) ns[k] = nsign[k] < 0 ? -1 : 1;
  int* d_ns = nullptr;
  double* d_out = nullptr;
  GBEM_CUDA(ctx, cudaMallocAsync(&d_ns, sizeof(int) * n, ctx->stream));
  GBEM_CUDA(ctx, cudaMallocAsync(&d_out, sizeof(double) * n, ctx->stream));
  GBEM_CUDA(ctx, cudaMemcpyAsync(d_ns, ns.data(), sizeof(int) * n, cudaMemcpyHostToDevice, ctx->stream));
  const unsigned ob = (unsigned)((npairs + kOracleWarps - 1) / kOracleWarps);
  k_st_oracle<<<ob, 32 * kOracleWarps, 0, ctx->stream>>>(ctx->d_panels, d_ns, (int)npairs, dbl ? 1 : 0, depth, d_out);
  GBEM_LAUNCH_CHECK(ctx);
  GBEM_CUDA(ctx, cudaMemcpyAsync(out, d_out, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  cudaFreeAsync(d_ns, ctx->stream);
  cudaFreeAsync(d_out, ctx->stream);
  GBEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return GBEM_OK;
}

int gbem_internal_selftest(gbem_ctx* ctx, int32_t pairs, uint64_t seed, const gbem_quad_config* cfg_in,
                           gbem_selftest_case* cases, int32_t* ncases) {
  if (pairs <= 0 || pairs > (1 << 22)) return ctx->fail(GBEM_EINVAL, "pairs per case must be in [1, 2^22]");
  if (!cases) return ctx->fail(GBEM_EINVAL, "null case array");
  gbem_quad_config cfg{};
  if (cfg_in) cfg = *cfg_in;
  const double rel_tol = cfg.rel_tol > 0 ? cfg.rel_tol : 1e-8;
  const int levels = cfg.max_levels > 0 ? cfg.max_levels : 16;
  const int64_t n2 = 2 * (int64_t)pairs;
  // the pairs live in the context's panel array (gbem_internal_pair_list reads them there)
  if (ctx->panel_cap < n2) {
    cudaFree(ctx->d_panels);
    ctx->d_panels = nullptr;
    ctx->panel_cap = 0;
    GBEM_CUDA(ctx, cudaMalloc(&ctx->d_panels, sizeof(DPanel) * (size_t)n2));
    ctx->panel_cap = n2;
  }
  int* d_ns = nullptr;
  double* d_buf = nullptr;
  unsigned long long* d_worst = nullptr;
  int32_t* d_conv = nullptr;
  GBEM_CUDA(ctx, cudaMalloc(&d_ns, sizeof(int) * pairs));
  GBEM_CUDA(ctx, cudaMalloc(&d_buf, sizeof(double) * 6 * (size_t)pairs));
  GBEM_CUDA(ctx, cudaMalloc(&d_conv, sizeof(int32_t) * pairs));
  GBEM_CUDA(ctx, cudaMalloc(&d_worst, sizeof(unsigned long long) * 10));
  GBEM_CUDA(ctx, cudaMemsetAsync(d_worst, 0, sizeof(unsigned long long) * 10, ctx->stream));
  double* semi = d_buf;
  double* o[3] = {d_buf + pairs, d_buf + 2 * (size_t)pairs, d_buf + 3 * (size_t)pairs};
  const unsigned gb = (unsigned)((pairs + 127) / 128), ob = (unsigned)((pairs + kOracleWarps - 1) / kOracleWarps);
  int rc = GBEM_OK;
  for (int c = 0; c < 10 && rc == GBEM_OK; ++c) {
    const CaseDef& cd = kCases[c];
    k_st_gen<<<gb, 128, 0, ctx->stream>>>(cd.gen, seed, pairs, ctx->d_panels, d_ns);
    GBEM_LAUNCH_CHECK(ctx);
    if (!cd.dbl) {
      gbem_quad_config q = cfg;
      rc = gbem_internal_pair_list(ctx, pairs, &q, semi, d_conv, nullptr);
      if (rc) break;
    } else {
      k_st_q<<<(unsigned)((pairs * 32 + 127) / 128), 128, 0, ctx->stream>>>(ctx->d_panels, d_ns, pairs, rel_tol,
                                                                            levels, semi);
      GBEM_LAUNCH_CHECK(ctx);
    }
    if (cd.mode == 1) {
      for (int k = 0; k < 3; ++k) {
        k_st_oracle<<<ob, 32 * kOracleWarps, 0, ctx->stream>>>(ctx->d_panels, d_ns, pairs, cd.dbl, 3 + k, o[k]);
        GBEM_LAUNCH_CHECK(ctx);
      }
    } else {
      k_st_oracle<<<ob, 32 * kOracleWarps, 0, ctx->stream>>>(ctx->d_panels, d_ns, pairs, cd.dbl,
                                                            cd.mode == 2 ? 3 : 6, o[2]);
      GBEM_LAUNCH_CHECK(ctx);
    }
    double* d_err = d_buf + 4 * (size_t)pairs;
    double* d_ref = d_buf + 5 * (size_t)pairs;
    k_st_worst<<<gb, 128, 0, ctx->stream>>>(semi, o[0], o[1], o[2], pairs, cd.mode, d_worst + c, d_err, d_ref);
    GBEM_LAUNCH_CHECK(ctx);
    // the worst pair of the class, for the report
    std::vector<double> herr((size_t)pairs);
    cudaError_t ce = cudaMemcpyAsync(herr.data(), d_err, sizeof(double) * pairs, cudaMemcpyDeviceToHost, ctx->stream);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(ctx->stream);
    if (ce != cudaSuccess) {
      rc = ctx->fail(GBEM_ECUDA, std::string("selftest: ") + cudaGetErrorString(ce));
      break;
    }
    int64_t arg = 0;
    for (int64_t k = 1; k < pairs; ++k)
      if (herr[(size_t)k] > herr[(size_t)arg]) arg = k;
    DPanel pt, ps;
    int ns = 0;
    double sv = 0, rv = 0;
    cudaMemcpy(&pt, ctx->d_panels + arg, sizeof(DPanel), cudaMemcpyDeviceToHost);
    cudaMemcpy(&ps, ctx->d_panels + pairs + arg, sizeof(DPanel), cudaMemcpyDeviceToHost);
    cudaMemcpy(&ns, d_ns + arg, sizeof(int), cudaMemcpyDeviceToHost);
    cudaMemcpy(&sv, semi + arg, sizeof(double), cudaMemcpyDeviceToHost);
    cudaMemcpy(&rv, d_ref + arg, sizeof(double), cudaMemcpyDeviceToHost);
    gbem_selftest_case& w = cases[c];
    const DPanel* pp[2] = {&pt, &ps};
    double* dst[2] = {w.worst_test, w.worst_source};
    for (int q = 0; q < 2; ++q) {
      dst[q][0] = pp[q]->axis;
      dst[q][1] = pp[q]->level;
      dst[q][2] = pp[q]->a0;
      dst[q][3] = pp[q]->a1;
      dst[q][4] = pp[q]->b0;
      dst[q][5] = pp[q]->b1;
    }
    w.worst_nsign = ns;
    w.worst_value = sv;
    w.worst_oracle = rv;
  }
  unsigned long long hw[10] = {};
  if (rc == GBEM_OK) {
    cudaError_t e = cudaMemcpyAsync(hw, d_worst, sizeof(hw), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = ctx->fail(GBEM_ECUDA, std::string("selftest: ") + cudaGetErrorString(e));
  }
  cudaFree(d_ns);
  cudaFree(d_buf);
  cudaFree(d_conv);
  cudaFree(d_worst);
  if (rc) return rc;
  for (int c = 0; c < 10; ++c) {
    gbem_selftest_case& out = cases[c];
    std::memset(out.name, 0, sizeof(out.name));
    std::strncpy(out.name, kCases[c].name, sizeof(out.name) - 1);
    out.pairs = pairs;
    double wv;
    std::memcpy(&wv, &hw[c], sizeof(wv));
    out.worst_rel = wv;
    out.tol = kCases[c].tol;
    out.pass = wv <= kCases[c].tol ? 1 : 0;
  }
  if (ncases) *ncases = 10;
  return GBEM_OK;
}

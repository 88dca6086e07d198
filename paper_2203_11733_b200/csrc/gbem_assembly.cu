// gbem_assembly.cu — Galerkin single-layer assembly on B200 (sm_100a).
//
// Replaces the reference's O(n^2/2) loop over u_pair_integral
// (proj/include/gbem/assembly.hpp:82-104, kernels.hpp:270-291).  Pipeline per
// chunk of upper-triangle tiles (32 x 32 pairs each):
//   1. k_classify<false>: per pair, gap/diameter test and class or far-field
//      Gauss orders; warp-aggregated (__match_any_sync) histogram over 2^16 keys.
//   2. k_scan: exclusive scan -> per-key queue segments.
//   3. k_classify<true>: fill the queue; pairs with equal keys are contiguous, so
//      every evaluation warp below runs one uniform loop structure.
//   4. k_far: anisotropic tensor Gauss-Legendre on 1/(4 pi r), one thread per
//      pair (FP64 pipe: DADD + MUFU.RSQ64H + 4 FP64 ops + DFMA per point).
//      k_coplanar: the reference's 16-corner closed form, one thread per pair.
//      k_near_warp: offset-parallel / orthogonal Romberg, one warp per pair.
//   5. k_symmetrize: mirror the lower triangle into the upper (tiled transpose).
// The matrix is column-major; entry (row j, col i), i <= j, is written at
// A[i*lda + j] so consecutive lanes (consecutive j) store contiguously.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "gbem_ctx.cuh"
#include "gbem_dmma_gemm.cuh"
#include "gbem_near.cuh"

using namespace gbem_gpu;

namespace gbem_gpu {
__constant__ double c_gx[kQMax + 1][kQMax];
__constant__ double c_gw[kQMax + 1][kQMax];
// c_delta[q]: far-field order q suffices along a direction of half-length h
// when gap >= c_delta[q] * h.  Derived from the Bernstein-ellipse bound of the
// end-on singularity, rho = 1 + d + sqrt(d (2 + d)), error ~ rho^(-2q);
// calibrated in tools/calib_far.c (far pairs have gap >= diam, so q <= 8 at
// far_tol = 1e-12).
__constant__ double c_delta[kQMax + 1];
// the same thresholds squared, in FP32, for the classifier: order q suffices when
// gap^2 / h^2 >= c_cd2f[q]
__constant__ float c_cd2f[kQMax + 1];
// Gauss-Legendre nodes / weights of the graded near-field rule (near_nodes(band) entries per band)
__constant__ double c_nx[kNearBands][48];
__constant__ double c_nw[kNearBands][48];
// list descriptor (type | (q1-1) << 2 | q2 << 5) -> index of its specialised
// far-field kernel (kFastDescs below), or -1
__constant__ __align__(16) int8_t c_fast_idx[512];
// Weight-folded nodes of the specialised far-field kernels: W / sqrt(x) = S / sqrt(x kappa)
// with kappa = (S / W)^2 a constant of the rule once the geometric scale S is factored out:
//   tent ramp of order q (S = h^2):      W_k = h^2 g_k (1 + x_k)   c_kr[q][k]  = 1 / (g_k (1 + x_k))^2
//   tent plateau of order q (S = h T):   W_k = h T g_k             c_kp[q][k]  = 1 / g_k^2
//   product rule q1 x q2 (S = h_I h_J):  W   = S g_a g_b           c_kpp[q1][q2][a q2 + b] = 1 / (g_a g_b)^2
constexpr int kQProd = 4;  // product inner lists up to 4 x 4
__constant__ double c_kr[kQMax + 1][kQMax];
__constant__ double c_kp[kQMax + 1][kQMax];
__constant__ double c_kpp[kQProd + 1][kQProd + 1][kQProd * kQProd];
}  // namespace gbem_gpu

namespace {

enum StatIdx {
  ST_NONCONV = 0,
  ST_NONFINITE,
  ST_NEAR_EVALS,
  ST_FAR_EVALS,
  ST_FAR_FLOPS,  // stored as double bits
  ST_COP,
  ST_PAR,
  ST_ORTH,
  ST_FAR,
  ST_FIRST_BAD,  // first (i << 32 | j) with a non-finite sample, ~0 if none
  ST_ROMB,       // near-contact pairs on the adaptive Romberg route
  ST_BAND0,      // .. ST_BAND0 + kNearBands - 1: graded Gauss-Legendre bands
  ST_COUNT = ST_BAND0 + 4
};

constexpr int kTile = 32;
constexpr int kClassifyThreads = 256;

// n-point Gauss-Legendre nodes (ascending) and weights on [-1, 1] (Newton on P_n).
void legendre_nodes(int q, double* gx, double* gw) {
  for (int i = 0; i < q; ++i) {
    long double x = cosl(3.14159265358979323846264338327950288L * (i + 0.75L) / (q + 0.5L));
    long double p0 = 1, p1 = x, dp = 1;
    for (int it = 0; it < 100; ++it) {
      p0 = 1;
      p1 = x;
      for (int k = 2; k <= q; ++k) {
        long double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      if (q == 1) {
        p1 = x;
        p0 = 1;
      }
      dp = q * (x * p1 - p0) / (x * x - 1);
      long double dx = p1 / dp;
      x -= dx;
      if (fabsl(dx) < 1e-19L) break;
    }
    p0 = 1;
    p1 = x;
    for (int k = 2; k <= q; ++k) {
      long double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    if (q == 1) {
      p1 = x;
      p0 = 1;
    }
    dp = q * (x * p1 - p0) / (x * x - 1);
    gx[q - 1 - i] = (double)x;
    gw[q - 1 - i] = (double)(2.0L / ((1.0L - x * x) * dp * dp));
  }
}

// Gauss-Legendre nodes on [-1, 1] by Newton on P_q.
void legendre_table(double gx[kQMax + 1][kQMax], double gw[kQMax + 1][kQMax]) {
  for (int q = 0; q <= kQMax; ++q)
    for (int k = 0; k < kQMax; ++k) gx[q][k] = gw[q][k] = 0.0;
  for (int q = 1; q <= kQMax; ++q) {
    for (int i = 0; i < q; ++i) {
      long double x = cosl(3.14159265358979323846264338327950288L * (i + 0.75L) / (q + 0.5L));
      long double p0 = 1, p1 = x, dp = 1;
      for (int it = 0; it < 100; ++it) {
        p0 = 1;
        p1 = x;
        for (int k = 2; k <= q; ++k) {
          long double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
          p0 = p1;
          p1 = p2;
        }
        if (q == 1) {
          p1 = x;
          p0 = 1;
        }
        dp = q * (x * p1 - p0) / (x * x - 1);
        long double dx = p1 / dp;
        x -= dx;
        if (fabsl(dx) < 1e-19L) break;
      }
      p0 = 1;
      p1 = x;
      for (int k = 2; k <= q; ++k) {
        long double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      if (q == 1) {
        p1 = x;
        p0 = 1;
      }
      dp = q * (x * p1 - p0) / (x * x - 1);
      // ascending nodes
      gx[q][q - 1 - i] = (double)x;
      gw[q][q - 1 - i] = (double)(2.0L / ((1.0L - x * x) * dp * dp));
    }
  }
}

// ---------------------------------------------------------------- classify

// Per-panel classification record, computed once per assembly (k_panel_cinfo):
// world extents (geometry.hpp:62-66), squared diameter (73), and 1 / h^2 of the
// two in-plane half-lengths for the far-field orders.  Every per-pair test is
// then done on squared distances (no sqrt / hypot per pair) and the orders in FP32.
struct __align__(16) CPanel {
  double lo[3], hi[3];
  double dm2;
  float iha2, ihb2;
  int axis, pad;
};

__global__ void k_panel_cinfo(const DPanel* __restrict__ P, int n, CPanel* __restrict__ out) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const DPanel p = P[k];
  CPanel c;
#pragma unroll
  for (int d = 0; d < 3; ++d) panel_extent(p, d, c.lo[d], c.hi[d]);
  const double la = p.a1 - p.a0, lb = p.b1 - p.b0;
  c.dm2 = la * la + lb * lb;
  c.iha2 = (float)(4.0 / (la * la));
  c.ihb2 = (float)(4.0 / (lb * lb));
  c.axis = p.axis;
  c.pad = 0;
  out[k] = c;
}

// far-field order along a direction from r2 = gap^2 / h^2: the smallest q with
// r2 >= c_cd2f[q] (thresholds decrease with q), i.e. 1 + #{k < kQMax : r2 < c_cd2f[k]}
// The same count for r2 = num / den without the division: r2 < t  <=>  num < t den (den > 0).
__device__ __forceinline__ int far_order_ratio(float num, float den) {
  const bool c4 = num < c_cd2f[4] * den;
  const bool c2 = num < (c4 ? c_cd2f[6] : c_cd2f[2]) * den;
  const bool c1 = num < (c4 ? (c2 ? c_cd2f[7] : c_cd2f[5]) : (c2 ? c_cd2f[3] : c_cd2f[1])) * den;
  return 1 + (c4 ? 4 : 0) + (c2 ? 2 : 0) + (c1 ? 1 : 0);
}

__device__ __forceinline__ int far_order_r2(float r2) {
  // q = 1 + #{k : r2 < c_cd2f[k]}; the thresholds decrease with k, so the count
  // is found by a three-level binary search
  const bool c4 = r2 < c_cd2f[4];
  const bool c2 = r2 < (c4 ? c_cd2f[6] : c_cd2f[2]);
  const bool c1 = r2 < (c4 ? (c2 ? c_cd2f[7] : c_cd2f[5]) : (c2 ? c_cd2f[3] : c_cd2f[1]));
  return 1 + (c4 ? 4 : 0) + (c2 ? 2 : 0) + (c1 ? 1 : 0);
}

// ---------------------------------------------------------------- far-field plan
//
// Difference-set quadrature.  The integrand of U = int_I int_J 1/(4 pi |x - y|)
// depends on x - y only, so along a world axis k that is in-plane for both
// panels the pair of 1-D integrals over [s0, s1] (I) and [u0, u1] (J) collapses
// to one integral over w = x_k - y_k with the trapezoidal weight
//   T(w) = |[s0, s1] ∩ [u0 + w, u1 + w]|   (ramp up, plateau, ramp down),
// the pushforward the reference applies analytically to offset-parallel pairs
// (kernels.hpp:96-125, tentSegments).  Each piece gets Gauss-Legendre of the
// order the far-field rule gives its half-length at the pair's gap; the plain
// product rule (q_I q_J nodes) is kept for an axis when it is cheaper.  An axis
// in-plane for one panel only contributes that panel's 1-D rule, the common
// normal of a parallel pair the constant offset.  A pair is three lists of
// (w_k, W_k), one per world axis, and
//   U = 1/(4 pi) sum_a sum_b sum_c W1_a W2_b W3_c / sqrt(w1_a^2 + w2_b^2 + w3_c^2):
// 95 nodes per far pair on config 2 instead of the 4-D tensor rule's 147
// (tools/calib_tent.c: worst relative error 2.2e-12 against a composite
// 3^4 x 12^4 truth over gap/diameter 1..32 at far_tol = 1e-12).
//
// The classifier decides the lists (orders in FP32 from the classification
// records) and packs them into a 31-bit plan stored beside the queue entry:
//   bit 0 orthogonal pair; bits 1 + 9 s .. 9 + 9 s: source list s as
//   type (2 bits) | q1 - 1 (3) | q2 (4); bits 28-29: source of the inner
//   (largest) list; bit 30: which of the two others is the middle one.
// Sources: parallel (shared axis ip0, shared axis ip1, normal offset);
// orthogonal (shared axis, I's rule along J's normal, J's rule along I's normal).
enum FarListType : int { kListConst = 0, kListSingle = 1, kListProduct = 2, kListTent = 3 };

// 1 / h^2 (FP32) of panel C's half-length along its in-plane world axis k
__device__ __forceinline__ float cp_ih2(const CPanel& C, int k) { return k == ip0(C.axis) ? C.iha2 : C.ihb2; }

// List descriptor of a shared in-plane axis k: tent or product, whichever has fewer nodes.
__device__ __forceinline__ uint32_t shared_axis_desc(const CPanel& A, const CPanel& B, int k, float g2, int& m) {
  const float ihA = cp_ih2(A, k), ihB = cp_ih2(B, k);
  const int qi = far_order_r2(g2 * ihA), qj = far_order_r2(g2 * ihB);
  const int qr = min(qi, qj);  // ramps: half-length min(L_I, L_J) / 2: the smaller panel's order
  const double Li = k == 0 ? A.hi[0] - A.lo[0] : (k == 1 ? A.hi[1] - A.lo[1] : A.hi[2] - A.lo[2]);
  const double Lj = k == 0 ? B.hi[0] - B.lo[0] : (k == 1 ? B.hi[1] - B.lo[1] : B.hi[2] - B.lo[2]);
  int qp = 0;
  if (Li != Lj) {
    const float dp = (float)fabs(Li - Lj);
    qp = far_order_ratio(4.0f * g2, dp * dp);  // half-length |L_I - L_J| / 2
  }
  if (2 * qr + qp < qi * qj) {
    m = 2 * qr + qp;
    return (uint32_t)kListTent | (uint32_t)(qr - 1) << 2 | (uint32_t)qp << 5;
  }
  m = qi * qj;
  return (uint32_t)kListProduct | (uint32_t)(qi - 1) << 2 | (uint32_t)qj << 5;
}

__device__ __forceinline__ uint32_t far_plan_code(const CPanel& A, const CPanel& B, float g2, const int8_t* fast_idx,
                                                  uint32_t& key) {
  uint32_t d[3];
  int m[3];
  const bool orth = A.axis != B.axis;
  if (!orth) {
    d[0] = shared_axis_desc(A, B, ip0(A.axis), g2, m[0]);
    d[1] = shared_axis_desc(A, B, ip1(A.axis), g2, m[1]);
    d[2] = kListConst;
    m[2] = 1;
  } else {
    d[0] = shared_axis_desc(A, B, 3 - A.axis - B.axis, g2, m[0]);
    const int qa = far_order_r2(g2 * cp_ih2(A, B.axis)), qb = far_order_r2(g2 * cp_ih2(B, A.axis));
    d[1] = (uint32_t)kListSingle | (uint32_t)(qa - 1) << 2;
    d[2] = (uint32_t)kListSingle | (uint32_t)(qb - 1) << 2;
    m[1] = qa;
    m[2] = qb;
  }
  // stable descending order of the sizes: inner source s0, then middle s1
  const int s0 = (m[0] >= m[1] && m[0] >= m[2]) ? 0 : (m[1] >= m[2] ? 1 : 2);
  const int r0 = s0 == 0 ? 1 : 0, r1 = s0 == 2 ? 1 : 2;  // remaining sources in index order
  const int mid_second = m[r1] > m[r0] ? 1 : 0;
  const int m1 = m[s0];
  const int m2 = mid_second ? m[r1] : m[r0];
  const int m3 = mid_second ? m[r0] : m[r1];
  // specialised kernels (k_far_orth / k_far_par) when the inner list has one of their descriptors
  const uint32_t di = s0 == 0 ? d[0] : (s0 == 1 ? d[1] : d[2]);
  const uint32_t dm = mid_second ? (r1 == 1 ? d[1] : d[2]) : (r0 == 0 ? d[0] : d[1]);
  const int fi = fast_idx[di];
  if (fi >= 0 && orth && s0 == 0) {
    key = kFastOrthBase + (uint32_t)(fi << 6 | (m2 - 1) << 3 | (m3 - 1));
  } else if (fi >= 0 && !orth && (dm & 3u) >= (uint32_t)kListProduct) {
    const uint32_t c2 = ((dm & 3u) == (uint32_t)kListTent ? 1u : 0u) | ((dm >> 2) & 7u) << 1 | (dm >> 5) << 4;
    key = kFastParBase + ((uint32_t)fi << 8 | c2);
  } else {
    key = far_key(m1, m2, m3);
  }
  return (orth ? 1u : 0u) | d[0] << 1 | d[1] << 10 | d[2] << 19 | (uint32_t)s0 << 28 | (uint32_t)mid_second << 30;
}

__device__ __forceinline__ uint32_t classify_pair(const CPanel& A, const CPanel& B, bool same, double near_ratio,
                                                  const int8_t* fast_idx, uint32_t& plan) {
  plan = 0;
  if (same) return kClsCoplanar;
  double gap2 = 0.0;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double g = fmax(fmax(B.lo[d] - A.hi[d], A.lo[d] - B.hi[d]), 0.0);
    gap2 = fma(g, g, gap2);
  }
  const double dm2 = fmax(A.dm2, B.dm2);
  const bool same_axis = A.axis == B.axis;
  if (gap2 < near_ratio * near_ratio * dm2) {
    if (same_axis && A.lo[A.axis] == B.lo[B.axis]) return kClsCoplanar;
    int band;
    if (gap2 == 0.0 || gap2 >= 1e-2 * dm2)  // gap >= 0.1 diam
      band = 0;
    else if (gap2 >= 4e-4 * dm2)  // 0.02
      band = 1;
    else if (gap2 >= 2.5e-5 * dm2)  // 0.005
      band = 2;
    else if (gap2 >= 1e-6 * dm2)  // 1e-3
      band = 3;
    else
      return same_axis ? kClsParallel : kClsOrthogonal;  // near contact: adaptive Romberg
    return (same_axis ? kClsParallelGL : kClsOrthogonalGL) + band;
  }
  uint32_t key;
  plan = far_plan_code(A, B, (float)gap2, fast_idx, key);
  return key;
}

// Per-CTA key aggregation: warp groups of equal keys (__match_any_sync) add
// their sizes into a shared open-addressing table; one global atomic per
// distinct key per CTA then counts (pass 1) or reserves the CTA's queue range
// (pass 2), and each warp group writes at range base + its offset.
constexpr int kHash = 1024;  // >= pairs per CTA: the table never fills
#ifndef GBEM_STAGE_MIN_KEYS
#define GBEM_STAGE_MIN_KEYS 40
#endif
constexpr int kStageMinKeys = GBEM_STAGE_MIN_KEYS;  // threads holding a used table slot above which the fill pass stages by key
constexpr uint32_t kEmpty = 0xFFFFFFFFu;

__device__ __forceinline__ int hash_slot(uint32_t* hkey, uint32_t key) {
  int s = (int)((key * 2654435761u) >> 22);  // 10 bits
  while (true) {
    const uint32_t prev = atomicCAS(&hkey[s], kEmpty, key);
    if (prev == kEmpty || prev == key) return s;
    s = (s + 1) & (kHash - 1);
  }
}

// One CTA per 32x32 tile of the upper triangle restricted to rows [rb, re)
// (full != 0: complete rows).  tile_row_off[r] = tiles in tile rows before r.
template <bool FILL>
__global__ void __launch_bounds__(kClassifyThreads)
    k_classify(const CPanel* __restrict__ P, int n, int rb, int re, int bi0, int nbt,
               const long long* __restrict__ tile_row_off, int nrows_t, long long tile_begin,
               double near_ratio, uint32_t* counts, uint32_t* cursors, uint64_t* queue, uint32_t* plans,
               uint64_t* kp, int full) {
  constexpr int kIter = kTile / (kClassifyThreads / 32);
  __shared__ CPanel si[kTile], sj[kTile];
  __shared__ uint32_t hkey[kHash], hcnt[kHash];
  __shared__ __align__(4) int8_t sfast[512];
  if (!FILL && threadIdx.x < 128)
    reinterpret_cast<uint32_t*>(sfast)[threadIdx.x] = reinterpret_cast<const uint32_t*>(c_fast_idx)[threadIdx.x];
  const long long t = tile_begin + blockIdx.x;
  // tile row of t: full rows hold nbt tiles each; upper-triangle rows hold
  // nbt - bi tiles, so tile_row_off[r] = r c - r (r - 1) / 2 with c = nbt - bi0,
  // inverted in closed form (a per-thread binary search over tile_row_off was
  // ~40% of the classifier's issue slots).  The fix-up loops only absorb the
  // rounding of the square root.
  int lo;
  if (full) {
    lo = (int)(t / nbt);
  } else {
    const double c2 = 2.0 * (nbt - bi0) + 1.0;
    lo = (int)((c2 - sqrt(fmax(c2 * c2 - 8.0 * (double)t, 0.0))) * 0.5);
    lo = min(max(lo, 0), nrows_t - 1);
    const long long c = nbt - bi0;
    auto off = [&](long long r) { return r * c - r * (r - 1) / 2; };
    while (lo > 0 && off(lo) > t) --lo;
    while (lo + 1 < nrows_t && off(lo + 1) <= t) ++lo;
  }
  const long long row_off = full ? (long long)lo * nbt : (long long)lo * (nbt - bi0) - (long long)lo * (lo - 1) / 2;
  const int bi = bi0 + lo;
  const int bj = (full ? 0 : bi) + (int)(t - row_off);  // full: whole rows (mirrored entries too)
  const int tid = threadIdx.x;
  if (!FILL && tid < kTile) {
    int i = bi * kTile + tid;
    if (i < n) si[tid] = P[i];
  } else if (!FILL && tid < 2 * kTile) {
    int j = bj * kTile + (tid - kTile);
    if (j < n) sj[tid - kTile] = P[j];
  }
  for (int s = tid; s < kHash; s += kClassifyThreads) {
    hkey[s] = kEmpty;
    hcnt[s] = 0;
  }
  __syncthreads();
  const int lane = tid & 31, warp = tid >> 5;
  const int j = bj * kTile + lane;
  uint32_t key[kIter], plan[kIter], leader_off[kIter];
  unsigned peers[kIter];
  int slot[kIter];
#pragma unroll
  for (int it = 0; it < kIter; ++it) {
    const int r = warp + it * (kClassifyThreads / 32);
    const int i = bi * kTile + r;
    const bool valid = i >= rb && i < re && j < n && (full || j >= i);
    // pass 1 classifies and keeps (key, plan) in tile order; pass 2 reads them back
    uint64_t* kp_at = kp + (size_t)blockIdx.x * (kTile * kTile) + r * kTile + lane;
    if (!FILL) {
      key[it] = valid ? classify_pair(si[r], sj[lane], i == j, near_ratio, sfast, plan[it]) : kEmpty;
      *kp_at = (uint64_t)key[it] << 32 | plan[it];
    } else {
      const uint64_t v = *kp_at;
      key[it] = (uint32_t)(v >> 32);
      plan[it] = (uint32_t)v;
    }
    peers[it] = __match_any_sync(0xffffffffu, key[it]);
    slot[it] = -1;
    leader_off[it] = 0;
    if (valid && lane == __ffs(peers[it]) - 1) {
      slot[it] = hash_slot(hkey, key[it]);
      leader_off[it] = atomicAdd(&hcnt[slot[it]], (uint32_t)__popc(peers[it]));
    }
  }
  __syncthreads();
  if constexpr (!FILL) {
    // one global atomic per distinct key of the tile
    for (int s = tid; s < kHash; s += kClassifyThreads) {
      const uint32_t k = hkey[s];
      if (k != kEmpty) atomicAdd(&counts[k], hcnt[s]);
    }
  } else {
    // The tile's entries are first grouped by key in shared memory (position = exclusive prefix of
    // the key's table slot + the warp group's offset + the lane's rank) and then written out in
    // that order, so consecutive threads store consecutive entries of one key's queue range: with
    // ~100 distinct keys per tile (config 5) a warp row holds 2-3 pairs per key, and storing from
    // the classification layout wrote 12 bytes into a separate 32-byte sector for almost every pair.
    __shared__ uint32_t slpre[kHash];
    __shared__ uint64_t s_entry[kTile * kTile];
    __shared__ uint32_t s_plan[kTile * kTile];
    __shared__ uint16_t s_slot[kTile * kTile];
    __shared__ uint32_t s_wsum[kClassifyThreads / 32];
    static_assert(kHash == 4 * kClassifyThreads, "four table slots per thread");
    uint32_t c[4], sum = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int sl = 4 * tid + q;
      const uint32_t k = hkey[sl];
      c[q] = k == kEmpty ? 0u : hcnt[sl];
      if (c[q]) hcnt[sl] = atomicAdd(&cursors[k], c[q]);  // hcnt becomes the key's range base for this tile
      sum += c[q];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += v;
    }
    if (lane == 31) s_wsum[warp] = incl;
    // few distinct keys in the tile (config 3: ~20): the classification layout already stores
    // long runs per key, and the staging pass would only cost (11.1 -> 12.3 ms on config 3)
    const int busy = __syncthreads_count(sum != 0);
    if (busy <= kStageMinKeys) {
#pragma unroll
      for (int it = 0; it < kIter; ++it) {
        if (key[it] == kEmpty) continue;
        const int leader = __ffs(peers[it]) - 1;
        uint32_t base = slot[it] >= 0 ? hcnt[slot[it]] + leader_off[it] : 0;
        base = __shfl_sync(peers[it], base, leader);
        const int r = warp + it * (kClassifyThreads / 32);
        const uint32_t rank = __popc(peers[it] & ((1u << lane) - 1u));
        queue[base + rank] = pack_entry((uint32_t)(bi * kTile + r), (uint32_t)j, key[it]);
        plans[base + rank] = plan[it];
      }
      return;
    }
    uint32_t wbase = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kClassifyThreads / 32; ++w) {
      if (w < warp) wbase += s_wsum[w];
      total += s_wsum[w];
    }
    uint32_t run = wbase + incl - sum;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      slpre[4 * tid + q] = run;
      run += c[q];
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kIter; ++it) {
      if (key[it] == kEmpty) continue;
      const int leader = __ffs(peers[it]) - 1;
      const int sl = __shfl_sync(peers[it], slot[it], leader);
      const uint32_t lo = __shfl_sync(peers[it], leader_off[it], leader);
      const int r = warp + it * (kClassifyThreads / 32);
      const uint32_t rank = __popc(peers[it] & ((1u << lane) - 1u));
      const uint32_t lpos = slpre[sl] + lo + rank;
      s_entry[lpos] = pack_entry((uint32_t)(bi * kTile + r), (uint32_t)j, key[it]);
      s_plan[lpos] = plan[it];
      s_slot[lpos] = (uint16_t)sl;
    }
    __syncthreads();
    for (uint32_t t2 = tid; t2 < total; t2 += kClassifyThreads) {
      const int sl = s_slot[t2];
      const uint32_t gpos = hcnt[sl] + (t2 - slpre[sl]);
      queue[gpos] = s_entry[t2];
      plans[gpos] = s_plan[t2];
    }
  }
}

// Warp-aggregated append of `key` (one atomic per distinct key in the warp),
// used by the pair-list mode.
template <bool FILL>
__device__ __forceinline__ void warp_append(bool valid, uint32_t key, uint32_t plan, uint32_t i, uint32_t j,
                                            uint32_t* counts, uint32_t* cursors, uint64_t* queue, uint32_t* plans) {
  unsigned active = __ballot_sync(0xffffffffu, valid);
  if (!valid) return;
  unsigned peers = __match_any_sync(active, key);
  int lane = threadIdx.x & 31;
  int leader = __ffs(peers) - 1;
  unsigned rank = __popc(peers & ((1u << lane) - 1u));
  uint32_t base = 0;
  if (lane == leader) {
    if (FILL)
      base = atomicAdd(&cursors[key], (uint32_t)__popc(peers));
    else
      atomicAdd(&counts[key], (uint32_t)__popc(peers));
  }
  if (FILL) {
    base = __shfl_sync(peers, base, leader);
    queue[base + rank] = pack_entry(i, j, key);
    plans[base + rank] = plan;
  }
}

// Pair-list mode: pair k is (panel k, panel npairs + k).
template <bool FILL>
__global__ void __launch_bounds__(256)
    k_classify_list(const CPanel* __restrict__ P, int npairs, double near_ratio, uint32_t* counts,
                    uint32_t* cursors, uint64_t* queue, uint32_t* plans) {
  __shared__ __align__(4) int8_t sfast[512];
  if (threadIdx.x < 128)
    reinterpret_cast<uint32_t*>(sfast)[threadIdx.x] = reinterpret_cast<const uint32_t*>(c_fast_idx)[threadIdx.x];
  __syncthreads();
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  bool valid = k < npairs;
  uint32_t key = 0, plan = 0;
  if (valid) key = classify_pair(P[k], P[npairs + k], false, near_ratio, sfast, plan);
  warp_append<FILL>(valid, key, plan, (uint32_t)k, (uint32_t)(npairs + k), counts, cursors, queue, plans);
}

// Exclusive scan of kNumKeys counts (one CTA of 1024 threads, 64 keys each);
// also seeds the fill cursors and accumulates the class totals into stats.
__global__ void __launch_bounds__(1024)
    k_scan(const uint32_t* __restrict__ counts, uint32_t* offsets, uint32_t* cursors,
           unsigned long long* stats) {
  __shared__ uint32_t part[1024];
  int t = threadIdx.x;
  constexpr int per = kNumKeys / 1024;
  // the thread's 64 counts as 16 independent 16-byte loads, all in flight at once
  static_assert(per == 64, "16 x uint4 per thread");
  uint4 cv[per / 4];
  const uint4* c4 = reinterpret_cast<const uint4*>(counts + t * per);
#pragma unroll
  for (int k = 0; k < per / 4; ++k) cv[k] = c4[k];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < per / 4; ++k) s += cv[k].x + cv[k].y + cv[k].z + cv[k].w;
  part[t] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    uint32_t v = t >= off ? part[t - off] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  uint32_t run = t ? part[t - 1] : 0;
  uint4* o4 = reinterpret_cast<uint4*>(offsets + t * per);
  uint4* u4 = reinterpret_cast<uint4*>(cursors + t * per);
#pragma unroll
  for (int k = 0; k < per / 4; ++k) {
    uint4 o;
    o.x = run;
    run += cv[k].x;
    o.y = run;
    run += cv[k].y;
    o.z = run;
    run += cv[k].z;
    o.w = run;
    run += cv[k].w;
    o4[k] = o;
    u4[k] = o;
  }
  if (t == 1023) offsets[kNumKeys] = run;
  if (t == 0) {
    unsigned long long par = counts[kClsParallel], orth = counts[kClsOrthogonal];
    for (int b = 0; b < kNearBands; ++b) {
      par += counts[kClsParallelGL + b];
      orth += counts[kClsOrthogonalGL + b];
    }
    atomicAdd(&stats[ST_COP], (unsigned long long)counts[kClsCoplanar]);
    atomicAdd(&stats[ST_PAR], par);
    atomicAdd(&stats[ST_ORTH], orth);
    atomicAdd(&stats[ST_ROMB], (unsigned long long)counts[kClsParallel] + counts[kClsOrthogonal]);
    for (int b = 0; b < kNearBands; ++b)
      atomicAdd(&stats[ST_BAND0 + b], (unsigned long long)counts[kClsParallelGL + b] + counts[kClsOrthogonalGL + b]);
  }
  __syncthreads();
  if (t == 0) {
    // far total = everything from kFarKeyBase on
    unsigned long long far = (unsigned long long)(offsets[kNumKeys] - offsets[kFarKeyBase]);
    atomicAdd(&stats[ST_FAR], far);
  }
}

// ---------------------------------------------------------------- evaluation

struct OutSpec {
  double* A;      // matrix mode (nullptr in list mode): entry (i, j) at A[i * lda + j * ldc]
  long long lda;
  long long ldc;
  double* out;    // list mode: out[i]
  int32_t* conv;  // list mode converged flags (may be null)
};

__device__ __forceinline__ double panel_area(const DPanel& p) { return (p.a1 - p.a0) * (p.b1 - p.b0); }

__device__ __forceinline__ void store_value(const OutSpec& o, uint32_t i, uint32_t j, const DPanel& Pi,
                                            const DPanel& Pj, double U) {
  if (o.A) {
    o.A[(long long)i * o.lda + (long long)j * o.ldc] = U / (panel_area(Pi) * panel_area(Pj));
  } else {
    o.out[i] = U;
  }
}

__device__ __forceinline__ double warp_reduce_d(double x) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
  return x;
}

// 1 / x: MUFU.RCP64H seed and two Newton steps (a few ulp; the far rule's own
// error is 1e-12), instead of an IEEE division's longer dependent sequence.
__device__ __forceinline__ double rcp64(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// acc + W y (3 - x y^2): twice W / sqrt(x) after one Newton step from the
// MUFU.RSQ64H seed y (relative error <= 9.1e-7; after the step <= 1.3e-12 per
// node, tools/rsq_acc.cu: an order below the far-field rule's own 1e-12
// tolerance and 100x inside the 1e-10 gate).  The factor 1/2 is applied once
// per pair.  With the DADD that forms x: DADD, DMUL, DFMA, DMUL, DFMA per node.
__device__ __forceinline__ double wrsq3_acc(double W, double x, double acc) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e3 = fma(-(x * y), y, 3.0);
  return fma(W * y, e3, acc);
}

// One decoded list: type, orders, and the geometry of its nodes
//   single:  w = p0 + p1 x_k,                  W = p1 g_k
//   product: w = p0 + p1 x_a - p2 x_b,         W = p1 g_a p2 g_b       (k = a q2 + b)
//   tent:    pieces [p0, p1] (T = w - p0), [p1, p2] (T = p4), [p2, p3] (T = p3 - w),
//            orders q1, q2, q1;  w = c + h x,  W = h g T(w)
//   const:   w = p0, W = 1
struct FarList {
  int type, q1, q2;
  double p0, p1, p2, p3, p4;
};

__device__ __forceinline__ void shared_axis_geom(const DPanel& A, const DPanel& B, int k, FarList& L) {
  double s0, s1, u0, u1;
  panel_extent(A, k, s0, s1);
  panel_extent(B, k, u0, u1);
  if (L.type == kListTent) {
    L.p0 = s0 - u1;
    L.p1 = fmin(s0 - u0, s1 - u1);
    L.p2 = fmax(s0 - u0, s1 - u1);
    L.p3 = s1 - u0;
    L.p4 = fmin(s1 - s0, u1 - u0);
  } else {
    L.p0 = 0.5 * (s0 + s1) - 0.5 * (u0 + u1);
    L.p1 = 0.5 * (s1 - s0);
    L.p2 = 0.5 * (u1 - u0);
  }
}

// List `src` (0..2) of a pair from its plan code and the panel records.
__device__ __forceinline__ void far_list(uint32_t code, int src, const DPanel& A, const DPanel& B, FarList& L) {
  const uint32_t d = (code >> (1 + 9 * src)) & 511u;
  L.type = (int)(d & 3u);
  L.q1 = (int)((d >> 2) & 7u) + 1;
  L.q2 = (int)(d >> 5);
  L.p0 = L.p1 = L.p2 = L.p3 = L.p4 = 0.0;
  const bool orth = code & 1u;
  if (src == 0) {
    shared_axis_geom(A, B, orth ? 3 - A.axis - B.axis : ip0(A.axis), L);
  } else if (!orth) {
    if (src == 1)
      shared_axis_geom(A, B, ip1(A.axis), L);
    else
      L.p0 = A.level - B.level;
  } else {
    // I's rule along J's normal (w = x - level_J), J's rule along I's normal
    const DPanel& C = src == 1 ? A : B;
    const DPanel& D = src == 1 ? B : A;
    double c0, c1;
    panel_extent(C, D.axis, c0, c1);
    L.p0 = 0.5 * (c0 + c1) - D.level;
    L.p1 = 0.5 * (c1 - c0);
  }
}

// A list's nodes into this thread's shared-memory slots (stride ST), walked
// piece by piece (one Gauss rule per piece: the panel rule of a single list,
// q_I shifted copies of the q_J rule for a product, ramp / plateau / ramp for
// a tent), so a node costs two table loads and four FP64 operations.
template <int ST>
__device__ __forceinline__ void emit_list(const FarList& L, const double* gx, const double* gw, double* w2,
                                          double* W) {
  if (L.type == kListTent) {
    int idx = 0;
    for (int piece = 0; piece < 3; ++piece) {
      const bool up = piece == 0, flat = piece == 1;
      const int q = flat ? L.q2 : L.q1;
      const double lo = up ? L.p0 : (flat ? L.p1 : L.p2), hi = up ? L.p1 : (flat ? L.p2 : L.p3);
      const double c = 0.5 * (lo + hi), h = 0.5 * (hi - lo);
      const double al = up ? -L.p0 : (flat ? L.p4 : L.p3), be = up ? 1.0 : (flat ? 0.0 : -1.0);
      for (int k = 0; k < q; ++k, ++idx) {
        const double w = fma(h, gx[q * kQMax + k], c);
        w2[idx * ST] = w * w;
        W[idx * ST] = (h * gw[q * kQMax + k]) * fma(be, w, al);
      }
    }
  } else if (L.type == kListProduct) {
    const int qi = L.q1, qj = L.q2;
    int idx = 0;
    for (int a = 0; a < qi; ++a) {
      const double ca = fma(L.p1, gx[qi * kQMax + a], L.p0);
      const double fa = (L.p1 * gw[qi * kQMax + a]) * L.p2;
      for (int bq = 0; bq < qj; ++bq, ++idx) {
        const double w = fma(-L.p2, gx[qj * kQMax + bq], ca);
        w2[idx * ST] = w * w;
        W[idx * ST] = fa * gw[qj * kQMax + bq];
      }
    }
  } else if (L.type == kListSingle) {
    const int q = L.q1;
    for (int k = 0; k < q; ++k) {
      const double w = fma(L.p1, gx[q * kQMax + k], L.p0);
      w2[k * ST] = w * w;
      W[k * ST] = L.p1 * gw[q * kQMax + k];
    }
  } else {
    w2[0] = L.p0 * L.p0;
    W[0] = 1.0;
  }
}

// Far field, one kernel per inner-list size M (the queue segment of keys with
// m1 = M).  Per pair: the plan written by the classifier names the three
// lists; the inner one (M nodes) goes to registers, the other two to
// per-thread shared-memory slots, then
//   for c < m3, b < m2:  acc += W3_c W2_b sum_a W1_a rsq64(w1_a^2 + w2_b^2 + w3_c^2)
// with (m2, m3) uniform across a warp (equal keys are contiguous).  Per node:
// DADD, MUFU.RSQ64H + Householder step (rsq64), DFMA.  OUT2 slots for the
// middle list (m2 <= m1 = M) and the smallest (m3 <= 8); CTAs of 128 threads
// (64 for M > 14, whose slots would not fit 48 KB).
__host__ __device__ constexpr int far_threads(int M) { return M <= 14 ? 128 : 64; }
template <int M>
#ifndef GBEM_FAR_MINB
#define GBEM_FAR_MINB 4  // CTAs per SM for M <= 12 (sweep tools/far_minb_ab.sh: 2, 3, 5, 6 are 24-43% slower)
#endif
__global__ void __launch_bounds__(far_threads(M), M <= 12 ? GBEM_FAR_MINB : 2)
    k_far(const DPanel* __restrict__ P, const uint64_t* __restrict__ queue, const uint32_t* __restrict__ plans,
          const uint32_t* __restrict__ offsets, OutSpec o, unsigned long long* stats) {
  constexpr int kFarThreads = far_threads(M);
  constexpr int OUT2 = M, OUT3 = M < 8 ? M : 8;
  __shared__ double sgx[(kQMax + 1) * kQMax], sgw[(kQMax + 1) * kQMax];
  __shared__ double ow2[(OUT2 + OUT3) * kFarThreads], oW[(OUT2 + OUT3) * kFarThreads];
  for (int t = threadIdx.x; t < (kQMax + 1) * kQMax; t += blockDim.x) {
    sgx[t] = (&c_gx[0][0])[t];
    sgw[t] = (&c_gw[0][0])[t];
  }
  __syncthreads();
  double* w2s = ow2 + threadIdx.x;  // middle list (and, first, the inner one): OUT2 = M slots
  double* W2s = oW + threadIdx.x;
  double* w3s = ow2 + OUT2 * kFarThreads + threadIdx.x;
  double* W3s = oW + OUT2 * kFarThreads + threadIdx.x;
  const uint32_t begin = offsets[far_key_first(M)];
  const uint32_t end = offsets[far_key_first(M + 1)];
  unsigned long long flops = 0, evals = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  // Software pipeline over a thread's pairs: the queue entry and plan two runs
  // ahead are loading, and the panel records of the next run are prefetched
  // into L1, while this pair is evaluated.
  uint32_t base = begin + (blockIdx.x * blockDim.x + (threadIdx.x & ~31u));
  uint32_t nidx = base + (threadIdx.x & 31u);
  uint64_t ne = nidx < end ? queue[nidx] : 0;
  uint32_t ncode = nidx < end ? plans[nidx] : 0;
  uint32_t nnidx = nidx + stride;
  uint64_t nne = nnidx < end ? queue[nnidx] : 0;
  uint32_t nncode = nnidx < end ? plans[nnidx] : 0;
  for (; base < end; base += stride) {
    const uint32_t idx = nidx;
    const uint64_t e = ne;
    const uint32_t code = ncode;
    nidx = nnidx;
    ne = nne;
    ncode = nncode;
    nnidx += stride;
    if (nnidx < end) {
      nne = queue[nnidx];
      nncode = plans[nnidx];
    }
    if (nidx < end) {
      asm volatile("prefetch.global.L1 [%0];" ::"l"(P + entry_i(ne)));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(P + entry_j(ne)));
    }
    if (idx >= end) continue;
    const uint32_t i = entry_i(e), j = entry_j(e), key = entry_key(e) - 16u;
    const int m2 = (int)((key >> 3) & 31u) + 1, m3 = (int)(key & 7u) + 1;
    const DPanel A = load_panel(P, i), B = load_panel(P, j);
    const int s0 = (int)((code >> 28) & 3u);
    const int r0 = s0 == 0 ? 1 : 0, r1 = s0 == 2 ? 1 : 2;
    const bool mid_second = (code >> 30) & 1u;
    double w1[M], W1[M];
#if defined(GBEM_FAR_SETUP_ONLY) && GBEM_FAR_SETUP_ONLY == 1  // timing: no list work at all
    for (int a = 0; a < M; ++a) w1[a] = W1[a] = A.a0 + B.b1 + code;
    w2s[0] = W2s[0] = w3s[0] = W3s[0] = 1.0;
    if (false)
#endif
    {
      // the inner list goes through the middle list's slots into registers
      // (a direct per-node register emission was 6% slower: code size)
      FarList L;
      far_list(code, s0, A, B, L);
      emit_list<kFarThreads>(L, sgx, sgw, w2s, W2s);
#pragma unroll
      for (int a = 0; a < M; ++a) {
        w1[a] = w2s[a * kFarThreads];
        W1[a] = W2s[a * kFarThreads];
      }
      far_list(code, mid_second ? r1 : r0, A, B, L);
      emit_list<kFarThreads>(L, sgx, sgw, w2s, W2s);
      far_list(code, mid_second ? r0 : r1, A, B, L);
      emit_list<kFarThreads>(L, sgx, sgw, w3s, W3s);
    }
    // the output scale now, so the panel records are dead during the node loop
    const double out_scale = 0.5 * (o.A ? rcp64(kFourPi * (panel_area(A) * panel_area(B))) : rcp64(kFourPi));
    double acc = 0.0;
#ifdef GBEM_FAR_SETUP_ONLY  // timing experiment: the per-pair setup without the node loop (results wrong)
    acc = w1[M - 1] + W1[M - 1] + w2s[0] + w3s[0];
    if (false)
#endif
    for (int c = 0; c < m3; ++c) {
      const double w3 = w3s[c * kFarThreads], W3 = W3s[c * kFarThreads];
      for (int b = 0; b < m2; ++b) {
        const double r2 = w3 + w2s[b * kFarThreads];
        // two partial sums break the FMA dependency chain
        double t0 = 0.0, t1 = 0.0;
#pragma unroll
        for (int a = 0; a < M; a += 2) {
          t0 = wrsq3_acc(W1[a], r2 + w1[a], t0);
          if (a + 1 < M) t1 = wrsq3_acc(W1[a + 1], r2 + w1[a + 1], t1);
        }
        acc = fma(W3 * W2s[b * kFarThreads], t0 + t1, acc);
      }
    }
    acc *= out_scale;  // 1/2 of the Newton step (wrsq3_acc), 1 / (4 pi area_I area_J)
    // counters in integer arithmetic (off the FP64 pipe)
    const uint32_t nodes = (uint32_t)(M * m2 * m3);
    evals += nodes;
    flops += 7u * nodes + 4u * (uint32_t)(m2 * m3) + 6u * (uint32_t)(M + m2 + m3) + 31u;  // per node: DADD, DMUL, DFMA, DMUL, DFMA
    if (o.A) {
      o.A[(long long)i * o.lda + (long long)j * o.ldc] = acc;
    } else {
      o.out[i] = acc;
      if (o.conv) o.conv[i] = 1;
    }
  }
  double fl = (double)flops, ev = (double)evals;
  fl = warp_reduce_d(fl);
  ev = warp_reduce_d(ev);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(reinterpret_cast<double*>(&stats[ST_FAR_FLOPS]), fl);
    atomicAdd(&stats[ST_FAR_EVALS], (unsigned long long)ev);
  }
}

// ---------------------------------------------------------------- far field, specialised
//
// Most far pairs share a handful of inner-list shapes (configs 2-4: 22
// descriptors cover 98%).  For those the generic kernel's per-pair setup --
// three descriptor decodes, three run-time emission loops through
// shared-memory slots and the reload of the inner list, more warp instructions
// than the node loops themselves (DESIGN 9) -- is replaced by kernels compiled
// per inner descriptor: the inner list is emitted straight into registers by
// fully unrolled code whose Gauss nodes are constant-bank operands, and the
// other two lists are never stored: the single rules of an orthogonal pair and
// the second shared axis of a parallel pair are generated inside the (c, b)
// loops (3-5 FP64 operations per M-node row).  The descriptor is part of the
// queue key, so a kernel's segment is contiguous and its loops warp-uniform.
#define GBEM_FAST_DESCS(X)                                                                              \
  X(0, kListProduct, 2, 2) X(1, kListProduct, 2, 3) X(2, kListProduct, 3, 2) X(3, kListProduct, 3, 3)     \
  X(4, kListTent, 3, 0) X(5, kListTent, 3, 1) X(6, kListTent, 3, 2) X(7, kListTent, 3, 3)                \
  X(8, kListTent, 3, 4) X(9, kListTent, 3, 5) X(10, kListTent, 4, 0) X(11, kListTent, 4, 1)              \
  X(12, kListTent, 4, 2) X(13, kListTent, 4, 3) X(14, kListTent, 4, 4) X(15, kListTent, 4, 5)            \
  X(16, kListTent, 5, 0) X(17, kListTent, 5, 1) X(18, kListTent, 5, 2) X(19, kListTent, 5, 3)            \
  X(20, kListTent, 5, 4) X(21, kListTent, 6, 0) X(22, kListTent, 6, 1) X(23, kListProduct, 2, 4)         \
  X(24, kListProduct, 4, 2)

__host__ __device__ constexpr int fast_inner_size(int type, int q1, int q2) {
  return type == kListTent ? 2 * q1 + q2 : q1 * q2;
}

// Inner list of a shared axis, I = [s0, s1], J = [u0, u1], into registers, weights folded into
// the nodes: slot k holds cw_k = w_k^2 kappa_k, so that inside the node loops
//   W_k / sqrt(r2 + w_k^2) = S / sqrt(fma(r2, kappa_k, cw_k))
// with kappa_k a constant-bank operand (c_kr / c_kp / c_kpp) and S one scale per piece.  Tent:
// ramps [p0, p0 + 2 hr] and [p3 - 2 hr, p3] (T = w - p0, p3 - w; hr = min(L_I, L_J) / 2, scale
// hr^2 in sr) around the plateau of half-length hp = |L_I - L_J| / 2 (T = 2 hr, scale 2 hr hp in
// sp); product: every node carries h_I h_J, which goes to `scale`.
template <int TYPE, int Q1, int Q2>
__device__ __forceinline__ void emit_inner(double s0, double s1, double u0, double u1,
                                           double (&cw)[fast_inner_size(TYPE, Q1, Q2)], double& sr, double& sp,
                                           double& scale) {
  if (TYPE == kListTent) {
    const double p0 = s0 - u1, p3 = s1 - u0;
    const double li = s1 - s0, lj = u1 - u0;
    const double hr = 0.5 * fmin(li, lj);
    sr = hr * hr;
    const double cu = p0 + hr, cd = p3 - hr;
#pragma unroll
    for (int k = 0; k < Q1; ++k) {
      const double w = fma(hr, c_gx[Q1][k], cu);
      cw[k] = (w * w) * c_kr[Q1][k];
    }
    if (Q2 > 0) {
      const double hp = 0.5 * fabs(li - lj), c = 0.5 * (p0 + p3);
      sp = (2.0 * hr) * hp;
#pragma unroll
      for (int k = 0; k < Q2; ++k) {
        const double w = fma(hp, c_gx[Q2][k], c);
        cw[Q1 + k] = (w * w) * c_kp[Q2][k];
      }
    }
#pragma unroll
    for (int k = 0; k < Q1; ++k) {
      const double w = fma(hr, c_gx[Q1][k], cd);
      cw[Q1 + Q2 + k] = (w * w) * c_kr[Q1][Q1 - 1 - k];  // T = hr (1 - x_k): the mirrored ramp
    }
  } else {
    const double p0 = 0.5 * (s0 + s1) - 0.5 * (u0 + u1), p1 = 0.5 * (s1 - s0), p2 = 0.5 * (u1 - u0);
    scale *= p1 * p2;
#pragma unroll
    for (int a = 0; a < Q1; ++a) {
      const double ca = fma(p1, c_gx[Q1][a], p0);
#pragma unroll
      for (int b = 0; b < Q2; ++b) {
        const double w = fma(-p2, c_gx[Q2][b], ca);
        cw[a * Q2 + b] = (w * w) * c_kpp[Q1][Q2][a * Q2 + b];
      }
    }
  }
}

// acc + 2 / sqrt(x): MUFU.RSQ64H seed and one Newton step, y (3 - x y^2) (the 1/2 is applied
// once per pair): DMUL, DFMA, DFMA -- with the DFMA that forms x, 4 FP64-pipe instructions per
// node beside the MUFU (wrsq3_acc, which carries a weight per node, needs 5).
__device__ __forceinline__ double rsq3_acc(double x, double acc) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return fma(y, fma(-(x * y), y, 3.0), acc);
}

// sum_k W_k * 2 / sqrt(r2 + w_k^2) over the inner list (weight-folded nodes, emit_inner)
template <int TYPE, int Q1, int Q2>
__device__ __forceinline__ double inner_row(const double (&cw)[fast_inner_size(TYPE, Q1, Q2)], double r2, double sr,
                                            double sp) {
  if (TYPE == kListTent) {
    double tu = 0.0, td = 0.0;
#pragma unroll
    for (int k = 0; k < Q1; ++k) {
      tu = rsq3_acc(fma(r2, c_kr[Q1][k], cw[k]), tu);
      td = rsq3_acc(fma(r2, c_kr[Q1][Q1 - 1 - k], cw[Q1 + Q2 + k]), td);
    }
    if (Q2 == 0) return sr * (tu + td);
    double tp = 0.0;
#pragma unroll
    for (int k = 0; k < Q2; ++k) tp = rsq3_acc(fma(r2, c_kp[Q2][k], cw[Q1 + k]), tp);
    return fma(sr, tu + td, sp * tp);
  } else {
    constexpr int M = Q1 * Q2;
    double t0 = 0.0, t1 = 0.0;
#pragma unroll
    for (int a = 0; a < M; a += 2) {
      t0 = rsq3_acc(fma(r2, c_kpp[Q1][Q2][a], cw[a]), t0);
      if (a + 1 < M) t1 = rsq3_acc(fma(r2, c_kpp[Q1][Q2][a + 1], cw[a + 1]), t1);
    }
    return t0 + t1;
  }
}

#ifndef GBEM_FAST_MINB
#define GBEM_FAST_MINB 4
#endif

// Orthogonal pairs: inner = the shared axis (descriptor TYPE, Q1, Q2), middle
// and outer = the single rules of orders m2 >= m3 (I along J's normal, J along
// I's normal; the plan's mid_second bit says which is the middle one).
template <int TYPE, int Q1, int Q2>
__global__ void __launch_bounds__(128, GBEM_FAST_MINB)
    k_far_orth(const DPanel* __restrict__ P, const uint64_t* __restrict__ queue, const uint32_t* __restrict__ plans,
               const uint32_t* __restrict__ offsets, OutSpec o, unsigned long long* stats, int d) {
  constexpr int M = fast_inner_size(TYPE, Q1, Q2);
  __shared__ double sgx[(kQMax + 1) * kQMax], sgw[(kQMax + 1) * kQMax];
  for (int t = threadIdx.x; t < (kQMax + 1) * kQMax; t += blockDim.x) {
    sgx[t] = (&c_gx[0][0])[t];
    sgw[t] = (&c_gw[0][0])[t];
  }
  __syncthreads();
  const uint32_t begin = offsets[kFastOrthBase + (uint32_t)(d << 6)];
  const uint32_t end = offsets[kFastOrthBase + (uint32_t)((d + 1) << 6)];
  unsigned long long flops = 0, evals = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  uint32_t base = begin + (blockIdx.x * blockDim.x + (threadIdx.x & ~31u));
  uint32_t nidx = base + (threadIdx.x & 31u);
  uint64_t ne = nidx < end ? queue[nidx] : 0;
  uint32_t ncode = nidx < end ? plans[nidx] : 0;
  uint32_t nnidx = nidx + stride;
  uint64_t nne = nnidx < end ? queue[nnidx] : 0;
  uint32_t nncode = nnidx < end ? plans[nnidx] : 0;
  DPanel nA = load_panel(P, nidx < end ? entry_i(ne) : 0u), nB = load_panel(P, nidx < end ? entry_j(ne) : 0u);
  for (; base < end; base += stride) {
    const uint32_t idx = nidx;
    const uint64_t e = ne;
    const uint32_t code = ncode;
    nidx = nnidx;
    ne = nne;
    ncode = nncode;
    nnidx += stride;
    if (nnidx < end) {
      nne = queue[nnidx];
      nncode = plans[nnidx];
    }
    // this pair's panel records were loaded during the previous pair's node loops
    // (an L1 prefetch covers one 128-byte line; 3 of 8 48-byte records straddle two)
    const DPanel A = nA, B = nB;
    if (nidx < end) {
      nA = load_panel(P, entry_i(ne));
      nB = load_panel(P, entry_j(ne));
    }
    if (idx >= end) continue;
    const uint32_t i = entry_i(e), j = entry_j(e), key = entry_key(e);
    const int m2 = (int)((key >> 3) & 7u) + 1, m3 = (int)(key & 7u) + 1;
    double scale = 0.5 * (o.A ? rcp64(kFourPi * (panel_area(A) * panel_area(B))) : rcp64(kFourPi));
    double cw[M], sr = 1.0, sp = 0.0;
    {
      double s0, s1, u0, u1;
      const int k = 3 - A.axis - B.axis;
      panel_extent(A, k, s0, s1);
      panel_extent(B, k, u0, u1);
      emit_inner<TYPE, Q1, Q2>(s0, s1, u0, u1, cw, sr, sp, scale);
    }
    // single rules: w = c + h x_k, W = h g_k (h folded into the scale)
    double c0, c1;
    panel_extent(A, B.axis, c0, c1);
    const double ca = 0.5 * (c0 + c1) - B.level, ha = 0.5 * (c1 - c0);
    panel_extent(B, A.axis, c0, c1);
    const double cb = 0.5 * (c0 + c1) - A.level, hb = 0.5 * (c1 - c0);
    scale *= ha * hb;
    const bool mid_second = (code >> 30) & 1u;
    const double cm = mid_second ? cb : ca, hm = mid_second ? hb : ha;
    const double co = mid_second ? ca : cb, ho = mid_second ? ha : hb;
    const double *gx2 = sgx + m2 * kQMax, *gw2 = sgw + m2 * kQMax;
    const double *gx3 = sgx + m3 * kQMax, *gw3 = sgw + m3 * kQMax;
    double acc = 0.0;
    for (int c = 0; c < m3; ++c) {
      const double w3 = fma(ho, gx3[c], co);
      const double w3s = w3 * w3, W3 = gw3[c];
      for (int b = 0; b < m2; ++b) {
        const double w2 = fma(hm, gx2[b], cm);
        acc = fma(W3 * gw2[b], inner_row<TYPE, Q1, Q2>(cw, fma(w2, w2, w3s), sr, sp), acc);
      }
    }
    acc *= scale;
    const uint32_t rows = (uint32_t)(m2 * m3);
    evals += (uint32_t)M * rows;
    flops += 7u * (uint32_t)M * rows + 7u * rows + 5u * (uint32_t)M + 40u;
    if (o.A) {
      o.A[(long long)i * o.lda + (long long)j * o.ldc] = acc;
    } else {
      o.out[i] = acc;
      if (o.conv) o.conv[i] = 1;
    }
  }
  double fl = (double)flops, ev = (double)evals;
  fl = warp_reduce_d(fl);
  ev = warp_reduce_d(ev);
  if ((threadIdx.x & 31) == 0 && ev > 0.0) {
    atomicAdd(reinterpret_cast<double*>(&stats[ST_FAR_FLOPS]), fl);
    atomicAdd(&stats[ST_FAR_EVALS], (unsigned long long)ev);
  }
}

// Parallel pairs: inner = the larger shared-axis list (descriptor TYPE, Q1, Q2;
// plan bits 28-29 say which in-plane axis), middle = the other shared axis,
// generated piece by piece inside the loop from the descriptor in the key;
// the normal offset is a constant.
template <int TYPE, int Q1, int Q2>
__global__ void __launch_bounds__(128, GBEM_FAST_MINB)
    k_far_par(const DPanel* __restrict__ P, const uint64_t* __restrict__ queue, const uint32_t* __restrict__ plans,
              const uint32_t* __restrict__ offsets, OutSpec o, unsigned long long* stats, int d) {
  constexpr int M = fast_inner_size(TYPE, Q1, Q2);
  __shared__ double sgx[(kQMax + 1) * kQMax], sgw[(kQMax + 1) * kQMax];
  for (int t = threadIdx.x; t < (kQMax + 1) * kQMax; t += blockDim.x) {
    sgx[t] = (&c_gx[0][0])[t];
    sgw[t] = (&c_gw[0][0])[t];
  }
  __syncthreads();
  const uint32_t begin = offsets[kFastParBase + (uint32_t)(d << 8)];
  const uint32_t end = offsets[kFastParBase + (uint32_t)((d + 1) << 8)];
  unsigned long long flops = 0, evals = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  uint32_t base = begin + (blockIdx.x * blockDim.x + (threadIdx.x & ~31u));
  uint32_t nidx = base + (threadIdx.x & 31u);
  uint64_t ne = nidx < end ? queue[nidx] : 0;
  uint32_t ncode = nidx < end ? plans[nidx] : 0;
  uint32_t nnidx = nidx + stride;
  uint64_t nne = nnidx < end ? queue[nnidx] : 0;
  uint32_t nncode = nnidx < end ? plans[nnidx] : 0;
  DPanel nA = load_panel(P, nidx < end ? entry_i(ne) : 0u), nB = load_panel(P, nidx < end ? entry_j(ne) : 0u);
  for (; base < end; base += stride) {
    const uint32_t idx = nidx;
    const uint64_t e = ne;
    const uint32_t code = ncode;
    nidx = nnidx;
    ne = nne;
    ncode = nncode;
    nnidx += stride;
    if (nnidx < end) {
      nne = queue[nnidx];
      nncode = plans[nnidx];
    }
    // this pair's panel records were loaded during the previous pair's node loops
    // (an L1 prefetch covers one 128-byte line; 3 of 8 48-byte records straddle two)
    const DPanel A = nA, B = nB;
    if (nidx < end) {
      nA = load_panel(P, entry_i(ne));
      nB = load_panel(P, entry_j(ne));
    }
    if (idx >= end) continue;
    const uint32_t i = entry_i(e), j = entry_j(e), key = entry_key(e);
    const bool tent2 = key & 1u;
    const int q1 = (int)((key >> 1) & 7u) + 1, q2 = (int)((key >> 4) & 15u);
    double scale = 0.5 * (o.A ? rcp64(kFourPi * (panel_area(A) * panel_area(B))) : rcp64(kFourPi));
    const bool inner_first = ((code >> 28) & 3u) == 0u;  // inner list on ip0, middle on ip1 (else swapped)
    double cw[M], sr = 1.0, sp = 0.0;
    {
      // a parallel pair's in-plane axes are the panels' own a / b spans
      const double s0 = inner_first ? A.a0 : A.b0, s1 = inner_first ? A.a1 : A.b1;
      const double u0 = inner_first ? B.a0 : B.b0, u1 = inner_first ? B.a1 : B.b1;
      emit_inner<TYPE, Q1, Q2>(s0, s1, u0, u1, cw, sr, sp, scale);
    }
    const double s0 = inner_first ? A.b0 : A.a0, s1 = inner_first ? A.b1 : A.a1;
    const double u0 = inner_first ? B.b0 : B.a0, u1 = inner_first ? B.b1 : B.a1;
    const double dz = A.level - B.level, dz2 = dz * dz;
    double acc = 0.0;
    int rows;
    if (tent2) {
      rows = 2 * q1 + q2;
      const double p0 = s0 - u1, p1 = fmin(s0 - u0, s1 - u1), p2 = fmax(s0 - u0, s1 - u1), p3 = s1 - u0;
      const double p4 = fmin(s1 - s0, u1 - u0);
      for (int piece = 0; piece < 3; ++piece) {
        const bool up = piece == 0, flat = piece == 1;
        const int q = flat ? q2 : q1;
        const double lo = up ? p0 : (flat ? p1 : p2), hi = up ? p1 : (flat ? p2 : p3);
        const double c = 0.5 * (lo + hi), h = 0.5 * (hi - lo);
        const double al = up ? -p0 : (flat ? p4 : p3), be = up ? 1.0 : (flat ? 0.0 : -1.0);
        const double *gx = sgx + q * kQMax, *gw = sgw + q * kQMax;
        for (int k = 0; k < q; ++k) {
          const double w = fma(h, gx[k], c);
          const double Wn = (h * gw[k]) * fma(be, w, al);
          acc = fma(Wn, inner_row<TYPE, Q1, Q2>(cw, fma(w, w, dz2), sr, sp), acc);
        }
      }
    } else {
      rows = q1 * q2;
      const double p0 = 0.5 * (s0 + s1) - 0.5 * (u0 + u1), p1 = 0.5 * (s1 - s0), p2 = 0.5 * (u1 - u0);
      scale *= p1 * p2;
      const double *gxa = sgx + q1 * kQMax, *gwa = sgw + q1 * kQMax;
      const double *gxb = sgx + q2 * kQMax, *gwb = sgw + q2 * kQMax;
      for (int a = 0; a < q1; ++a) {
        const double ca = fma(p1, gxa[a], p0), fa = gwa[a];
        for (int b = 0; b < q2; ++b) {
          const double w = fma(-p2, gxb[b], ca);
          acc = fma(fa * gwb[b], inner_row<TYPE, Q1, Q2>(cw, fma(w, w, dz2), sr, sp), acc);
        }
      }
    }
    acc *= scale;
    evals += (uint32_t)(M * rows);
    flops += 7u * (uint32_t)(M * rows) + 8u * (uint32_t)rows + 5u * (uint32_t)M + 40u;
    if (o.A) {
      o.A[(long long)i * o.lda + (long long)j * o.ldc] = acc;
    } else {
      o.out[i] = acc;
      if (o.conv) o.conv[i] = 1;
    }
  }
  double fl = (double)flops, ev = (double)evals;
  fl = warp_reduce_d(fl);
  ev = warp_reduce_d(ev);
  if ((threadIdx.x & 31) == 0 && ev > 0.0) {
    atomicAdd(reinterpret_cast<double*>(&stats[ST_FAR_FLOPS]), fl);
    atomicAdd(&stats[ST_FAR_EVALS], (unsigned long long)ev);
  }
}

__global__ void __launch_bounds__(128)
    k_coplanar(const DPanel* __restrict__ P, const uint64_t* __restrict__ queue,
               const uint32_t* __restrict__ offsets, OutSpec o) {
  const uint32_t begin = offsets[kClsCoplanar], end = offsets[kClsCoplanar + 1];
  for (uint32_t idx = begin + blockIdx.x * blockDim.x + threadIdx.x; idx < end;
       idx += gridDim.x * blockDim.x) {
    uint64_t e = queue[idx];
    uint32_t i = entry_i(e), j = entry_j(e);
    DPanel Pi = load_panel(P, i), Pj = load_panel(P, j);
    // canonical order (kernels.hpp:273-274) so the value matches the reference's rounding
    const DPanel& a = d_rect_less(Pj, Pi) ? Pj : Pi;
    const DPanel& b = d_rect_less(Pj, Pi) ? Pi : Pj;
    double U = d_u_coplanar(a.a0, a.a1, a.b0, a.b1, b.a0, b.a1, b.b0, b.b1);
    store_value(o, i, j, Pi, Pj, U);
    if (!o.A && o.conv) o.conv[i] = 1;
  }
}

// Graded Gauss-Legendre near field (keys 2..9): a team of kNearTeam lanes
// per pair shares its quadrature nodes (gl_graded), partial sums folded by
// shuffles in a fixed order; the queue is sorted by band, so a warp's teams
// mostly run the same node counts.
__global__ void __launch_bounds__(128)
    k_near_gl(const DPanel* __restrict__ P, const uint64_t* __restrict__ queue,
              const uint32_t* __restrict__ offsets, OutSpec o, unsigned long long* stats) {
  const uint32_t begin = offsets[kClsParallelGL], end = offsets[kClsOrthogonalGL + kNearBands];
  const int tl = threadIdx.x % kNearTeam;
  long long evals = 0, nonfinite = 0;
  const uint32_t team = (blockIdx.x * blockDim.x + threadIdx.x) / kNearTeam;
  const uint32_t nteams = gridDim.x * blockDim.x / kNearTeam;
  // trip count uniform across the warp (inactive teams run with a dummy pair)
  const uint32_t warp_team0 = team - (threadIdx.x % 32) / kNearTeam;
  for (uint32_t base = begin + warp_team0; base < end; base += nteams) {
    const uint32_t idx = base + (threadIdx.x % 32) / kNearTeam;
    const bool active = idx < end;
    uint64_t e = queue[active ? idx : base];
    uint32_t i = entry_i(e), j = entry_j(e), key = entry_key(e);
    DPanel Pi = load_panel(P, i), Pj = load_panel(P, j);
    bool swap = d_rect_less(Pj, Pi);
    const DPanel& a = swap ? Pj : Pi;
    const DPanel& b = swap ? Pi : Pj;
    bool bad = false;
    const bool par = key < (uint32_t)kClsOrthogonalGL;
    const int band = (int)key - (par ? kClsParallelGL : kClsOrthogonalGL);
    double U = par ? gl_u_parallel(a, b, band, c_nx, c_nw, bad, tl)
                   : gl_u_orthogonal(a, b, band, c_nx, c_nw, bad, tl);
    int bb = bad ? 1 : 0;
#pragma unroll
    for (int off = 1; off < kNearTeam; off <<= 1) {
      U += __shfl_xor_sync(0xffffffffu, U, off);
      bb |= __shfl_xor_sync(0xffffffffu, bb, off);
    }
    bad = bb != 0;
    if (active && tl == 0) {
      evals += 2 * near_nodes(band);
      store_value(o, i, j, Pi, Pj, U);
      if (!o.A && o.conv) o.conv[i] = 1;
      if (bad) {
        ++nonfinite;
        atomicMin(&stats[ST_FIRST_BAD], ((unsigned long long)i << 32) | j);
      }
    }
  }
  if (nonfinite) atomicAdd(&stats[ST_NONFINITE], (unsigned long long)nonfinite);
  if (evals) atomicAdd(&stats[ST_NEAR_EVALS], (unsigned long long)evals);
}

// Near-contact pairs are few (42 of 2.5e9 in a config-5 row chunk) and slow (the adaptive Romberg of
// one pair keeps a warp busy for 1-4 ms), so a kernel over one chunk's pairs is a 1-4 ms launch that
// occupies two or three warps.  The chunks of an assembly therefore only collect them
// (k_romb_collect moves the chunk's Romberg-route queue entries to a list that persists over the
// chunks) and one k_near_warp launch at the end evaluates the whole list, one warp per pair.  What does
// not fit the list is evaluated in place (skip = the number taken from this chunk).
constexpr uint32_t kRombCap = 1u << 20;

__global__ void __launch_bounds__(256)
    k_romb_collect(const uint64_t* __restrict__ queue, const uint32_t* __restrict__ offsets, uint64_t* list,
                   uint32_t* cnt) {
  const uint32_t begin = offsets[kClsParallel], end = offsets[kClsOrthogonal + 1];  // keys 10, 11
  __shared__ uint32_t s_base, s_take;
  if (threadIdx.x == 0) {  // one CTA, launches ordered on their stream
    s_base = cnt[0];
    s_take = min(end - begin, kRombCap - s_base);
    cnt[0] = s_base + s_take;
    cnt[1] = s_take;
  }
  __syncthreads();
  for (uint32_t k = threadIdx.x; k < s_take; k += blockDim.x) list[s_base + k] = queue[begin + k];
}

// list_cnt == nullptr: the Romberg-route entries of the queue, from `skip` entries in (nullptr: 0);
// else queue is the collected list of *list_cnt entries.
__global__ void __launch_bounds__(128)
    k_near_warp(const DPanel* __restrict__ P, const uint64_t* __restrict__ queue,
                const uint32_t* __restrict__ offsets, OutSpec o, double rel_tol, int max_levels,
                unsigned long long* stats, const uint32_t* skip = nullptr, const uint32_t* list_cnt = nullptr) {
  const uint32_t begin = list_cnt ? 0u : offsets[kClsParallel] + (skip ? *skip : 0u);
  const uint32_t end = list_cnt ? *list_cnt : offsets[kClsOrthogonal + 1];
  if (begin >= end) return;
  const int lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  long long evals = 0;
  for (uint32_t idx = begin + warp; idx < end; idx += nwarps) {
    uint64_t e = queue[idx];
    uint32_t i = entry_i(e), j = entry_j(e), key = entry_key(e);
    DPanel Pi = load_panel(P, i), Pj = load_panel(P, j);
    bool swap = d_rect_less(Pj, Pi);
    const DPanel& a = swap ? Pj : Pi;
    const DPanel& b = swap ? Pi : Pj;
    WarpQuad st;
    double U = key == kClsParallel ? warp_u_parallel(a, b, rel_tol, max_levels, lane, st)
                                   : warp_u_orthogonal(a, b, rel_tol, max_levels, lane, st);
    evals += st.evals;
    if (lane == 0) {
      store_value(o, i, j, Pi, Pj, U);
      if (!o.A && o.conv) o.conv[i] = st.converged ? 1 : 0;
      if (!st.converged) atomicAdd(&stats[ST_NONCONV], 1ull);
      if (st.nonfinite) {
        atomicAdd(&stats[ST_NONFINITE], 1ull);
        atomicMin(&stats[ST_FIRST_BAD], ((unsigned long long)i << 32) | j);
      }
    }
  }
  if (lane == 0) atomicAdd(&stats[ST_NEAR_EVALS], (unsigned long long)evals);
}

// Mirror A[i*lda + j] (j >= i) into A[j*lda + i] over 32x32 tiles (bi <= bj).
// 64 x 64 tiles, 16 loads per thread issued before any store (32 KB per CTA in
// flight, 6 CTAs per SM), transposed through shared memory.
constexpr int kSymTile = 64;
__global__ void __launch_bounds__(256) k_symmetrize(double* A, long long lda, int n, int nbt) {
  constexpr int TS = kSymTile, RPT = TS * TS / 256 / 2;  // rows per thread per half-tile column
  __shared__ double tile[TS][TS + 1];
  // linear upper-triangle tile index -> (bi, bj)
  long long t = blockIdx.x;
  int bi = (int)floor((2.0 * nbt + 1.0 - sqrt((2.0 * nbt + 1.0) * (2.0 * nbt + 1.0) - 8.0 * (double)t)) / 2.0);
  auto rowoff = [nbt](long long b) { return b * nbt - b * (b - 1) / 2; };
  while (bi > 0 && rowoff(bi) > t) --bi;
  while (rowoff(bi + 1) <= t) ++bi;
  const int bj = bi + (int)(t - rowoff(bi));
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 warps
  double v[RPT][2];
#pragma unroll
  for (int u = 0; u < RPT; ++u)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = ty + 8 * u, i = bi * TS + r, j = bj * TS + h * 32 + tx;
      v[u][h] = (i < n && j < n && j >= i) ? A[(long long)i * lda + j] : 0.0;
    }
#pragma unroll
  for (int u = 0; u < RPT; ++u)
#pragma unroll
    for (int h = 0; h < 2; ++h) tile[ty + 8 * u][h * 32 + tx] = v[u][h];
  __syncthreads();
#pragma unroll
  for (int u = 0; u < RPT; ++u)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = ty + 8 * u, j = bj * TS + r, i = bi * TS + h * 32 + tx;
      if (i < n && j < n && j > i) A[(long long)j * lda + i] = tile[h * 32 + tx][r];
    }
}

__global__ void k_pack_panels(const uint8_t* axis, const double* level, const double* a0,
                              const double* a1, const double* b0, const double* b1, int n,
                              DPanel* out) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  DPanel p;
  p.level = level[k];
  p.a0 = a0[k];
  p.a1 = a1[k];
  p.b0 = b0[k];
  p.b1 = b1[k];
  p.axis = axis[k];
  p.pad = 0;
  out[k] = p;
}

int grow(gbem_ctx* ctx, void** p, size_t bytes_needed, int64_t* cap_elems, size_t elem) {
  if ((size_t)*cap_elems * elem >= bytes_needed && *p) return GBEM_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  cudaError_t e = cudaMalloc(p, bytes_needed);
  if (e != cudaSuccess) {
    *cap_elems = 0;
    return ctx->fail(GBEM_ECUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  }
  *cap_elems = (int64_t)(bytes_needed / elem);
  return GBEM_OK;
}

// Classification records of the n resident panels (k_panel_cinfo).
int prepare_cinfo(gbem_ctx* ctx, int64_t n) {
  int rc = grow(ctx, &ctx->d_cinfo, sizeof(CPanel) * (size_t)n, &ctx->cinfo_cap, sizeof(CPanel));
  if (rc) return rc;
  k_panel_cinfo<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(ctx->d_panels, (int)n,
                                                                     (CPanel*)ctx->d_cinfo);
  GBEM_LAUNCH_CHECK(ctx);
  return GBEM_OK;
}

int prepare_work(gbem_ctx* ctx, const gbem_quad_config* cfg_in, gbem_quad_config* cfg) {
  gbem_quad_config c{};
  if (cfg_in) c = *cfg_in;
  if (!(c.rel_tol > 0)) c.rel_tol = 1e-8;
  if (c.max_levels <= 0) c.max_levels = 16;
  if (c.max_levels > kRombMax) return ctx->fail(GBEM_EINVAL, "max_levels exceeds 20");
  if (!(c.near_ratio > 0)) c.near_ratio = 1.0;
  if (c.near_ratio < 1.0) return ctx->fail(GBEM_EINVAL, "near_ratio must be >= 1 (far-field orders are capped at 8)");
  if (!(c.far_tol > 0)) c.far_tol = 1e-12;
  *cfg = c;
  if (!ctx->d_counts) {
    GBEM_CUDA(ctx, cudaMalloc(&ctx->d_counts, sizeof(uint32_t) * kNumKeys));
    GBEM_CUDA(ctx, cudaMalloc(&ctx->d_offsets, sizeof(uint32_t) * (kNumKeys + 1)));
    GBEM_CUDA(ctx, cudaMalloc(&ctx->d_cursors, sizeof(uint32_t) * kNumKeys));
    GBEM_CUDA(ctx, cudaMalloc(&ctx->d_stats, sizeof(unsigned long long) * ST_COUNT));
    GBEM_CUDA(ctx, cudaMallocHost(&ctx->h_stats, sizeof(unsigned long long) * ST_COUNT));
  }
  // far-field order thresholds
  double delta[kQMax + 1];
  delta[0] = 1e300;
  for (int q = 1; q <= kQMax; ++q) {
    double rho = std::pow(c.far_tol, -1.0 / (2.0 * q));
    delta[q] = 0.5 * (rho + 1.0 / rho) - 1.0;
  }
  GBEM_CUDA(ctx, cudaMemcpyToSymbolAsync(c_delta, delta, sizeof(delta), 0, cudaMemcpyHostToDevice,
                                         ctx->stream));
  float cd2f[kQMax + 1];
  cd2f[0] = 3.0e38f;
  for (int q = 1; q <= kQMax; ++q) cd2f[q] = (float)(delta[q] * delta[q]);
  GBEM_CUDA(ctx, cudaMemcpyToSymbolAsync(c_cd2f, cd2f, sizeof(cd2f), 0, cudaMemcpyHostToDevice, ctx->stream));
  GBEM_CUDA(ctx, cudaMemsetAsync(ctx->d_stats, 0, sizeof(unsigned long long) * ST_COUNT, ctx->stream));
  // ST_FIRST_BAD starts at ~0 (atomicMin target)
  GBEM_CUDA(ctx, cudaMemsetAsync(ctx->d_stats + ST_FIRST_BAD, 0xFF, sizeof(unsigned long long), ctx->stream));
  return GBEM_OK;
}

// Evaluate every queued class for the current chunk.
int run_eval(gbem_ctx* ctx, const OutSpec& o, const gbem_quad_config& cfg, float* ms_far,
             float* ms_near, bool defer_romberg = false) {
  int sms = ctx->num_sms;
  // The near-field kernels (closed-form coplanar, graded Gauss-Legendre, warp Romberg) write
  // entries no far-field kernel touches and are latency-bound -- a chunk's handful of
  // near-contact pairs keeps one warp each busy for ~1 ms in k_near_warp -- so they run on a
  // second stream beside the far-field kernels (config 5: near 588 of 2,690 ms when serial).
  // With per-phase timing requested the phases run one after the other, as their times are defined.
  static const bool near_serial = getenv("GBEM_NEAR_SERIAL") != nullptr;
  const bool overlap = !ms_far && !ms_near && !near_serial;
  cudaStream_t ns = ctx->stream;
  if (overlap) {
    if (!ctx->near_stream) {
      GBEM_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->near_stream, cudaStreamNonBlocking));
      GBEM_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_near_fork, cudaEventDisableTiming));
      GBEM_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_near_join, cudaEventDisableTiming));
    }
    ns = ctx->near_stream;
    GBEM_CUDA(ctx, cudaEventRecord(ctx->ev_near_fork, ctx->stream));
    GBEM_CUDA(ctx, cudaStreamWaitEvent(ns, ctx->ev_near_fork, 0));
  }
  // The ~75 far-field kernels of a chunk (one per inner-list descriptor / size) write disjoint
  // entries; most are small, and run one after the other each pays its launch gap and the tail
  // where its last CTAs drain.  Dealt round robin over four streams the tails fill with the next
  // kernels' CTAs.
  static const int far_nstreams = getenv("GBEM_FAR_STREAMS") ? std::max(1, std::min(1 + gbem_ctx::kFarStreams, atoi(getenv("GBEM_FAR_STREAMS")))) : 1 + gbem_ctx::kFarStreams;
  const int nfs = overlap ? far_nstreams : 1;
  cudaStream_t fs[1 + gbem_ctx::kFarStreams];
  fs[0] = ctx->stream;
  for (int k = 1; k < nfs; ++k) {
    if (!ctx->far_stream[k - 1]) {
      GBEM_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->far_stream[k - 1], cudaStreamNonBlocking));
      GBEM_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_far_join[k - 1], cudaEventDisableTiming));
    }
    fs[k] = ctx->far_stream[k - 1];
    GBEM_CUDA(ctx, cudaStreamWaitEvent(fs[k], ctx->ev_near_fork, 0));
  }
  int far_rr = 0;
#define GBEM_FS (fs[far_rr++ % nfs])
  static const int near_skip = getenv("GBEM_DBG_SKIP_NEAR") ? atoi(getenv("GBEM_DBG_SKIP_NEAR")) : 0;  // timing experiments
  auto near_kernels = [&]() -> int {
    if (near_skip == 3) return GBEM_OK;
    // the longest-running kernel first
    if (defer_romberg && near_skip != 1) {
      k_romb_collect<<<1, 256, 0, ns>>>(ctx->d_queue, ctx->d_offsets, ctx->d_romb, ctx->d_romb_cnt);
      GBEM_LAUNCH_CHECK(ctx);
    }
    if (near_skip != 1)
      k_near_warp<<<sms * 8, 128, 0, ns>>>(ctx->d_panels, ctx->d_queue, ctx->d_offsets, o, cfg.rel_tol,
                                           cfg.max_levels, ctx->d_stats, defer_romberg ? ctx->d_romb_cnt + 1 : nullptr);
    GBEM_LAUNCH_CHECK(ctx);
    k_near_gl<<<sms * 8, 128, 0, ns>>>(ctx->d_panels, ctx->d_queue, ctx->d_offsets, o, ctx->d_stats);
    GBEM_LAUNCH_CHECK(ctx);
    k_coplanar<<<sms * 4, 128, 0, ns>>>(ctx->d_panels, ctx->d_queue, ctx->d_offsets, o);
    GBEM_LAUNCH_CHECK(ctx);
    return GBEM_OK;
  };
  if (overlap) {
    if (int rc = near_kernels()) return rc;
    GBEM_CUDA(ctx, cudaEventRecord(ctx->ev_near_join, ns));
  }
  cudaEventRecord(ctx->ev[2], ctx->stream);
#define GBEM_FAR(M) \
  k_far<M><<<sms * 4, far_threads(M), 0, GBEM_FS>>>(ctx->d_panels, ctx->d_queue, ctx->d_plan, \
                                                                     ctx->d_offsets, o, ctx->d_stats); \
  GBEM_LAUNCH_CHECK(ctx);
  GBEM_FAR(1) GBEM_FAR(2) GBEM_FAR(3) GBEM_FAR(4) GBEM_FAR(5) GBEM_FAR(6) GBEM_FAR(7) GBEM_FAR(8)
  GBEM_FAR(9) GBEM_FAR(10) GBEM_FAR(11) GBEM_FAR(12) GBEM_FAR(13) GBEM_FAR(14) GBEM_FAR(15) GBEM_FAR(16)
  GBEM_FAR(17) GBEM_FAR(18) GBEM_FAR(19) GBEM_FAR(20) GBEM_FAR(21) GBEM_FAR(22) GBEM_FAR(23) GBEM_FAR(24)
#undef GBEM_FAR
#define GBEM_FAST(D, TYPE, Q1, Q2)                                                                                \
  k_far_orth<TYPE, Q1, Q2><<<sms * GBEM_FAST_MINB, 128, 0, GBEM_FS>>>(ctx->d_panels, ctx->d_queue, ctx->d_plan, \
                                                                         ctx->d_offsets, o, ctx->d_stats, D);      \
  GBEM_LAUNCH_CHECK(ctx);                                                                                         \
  k_far_par<TYPE, Q1, Q2><<<sms * GBEM_FAST_MINB, 128, 0, GBEM_FS>>>(ctx->d_panels, ctx->d_queue, ctx->d_plan,  \
                                                                        ctx->d_offsets, o, ctx->d_stats, D);       \
  GBEM_LAUNCH_CHECK(ctx);
  GBEM_FAST_DESCS(GBEM_FAST)
#undef GBEM_FAST
#undef GBEM_FS
  for (int k = 1; k < nfs; ++k) {
    GBEM_CUDA(ctx, cudaEventRecord(ctx->ev_far_join[k - 1], fs[k]));
    GBEM_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_far_join[k - 1], 0));
  }
  cudaEventRecord(ctx->ev[3], ctx->stream);
  if (overlap) {
    GBEM_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_near_join, 0));
  } else {
    if (int rc = near_kernels()) return rc;
  }
  cudaEventRecord(ctx->ev[4], ctx->stream);
  if (ms_far || ms_near) {
    GBEM_CUDA(ctx, cudaEventSynchronize(ctx->ev[4]));
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, ctx->ev[2], ctx->ev[3]);
    cudaEventElapsedTime(&b, ctx->ev[3], ctx->ev[4]);
    if (ms_far) *ms_far += a;
    if (ms_near) *ms_near += b;
  }
  return GBEM_OK;
}

int finish_stats(gbem_ctx* ctx, gbem_assembly_stats* stats, int64_t pairs_total) {
  GBEM_CUDA(ctx, cudaMemcpyAsync(ctx->h_stats, ctx->d_stats, sizeof(unsigned long long) * ST_COUNT,
                                 cudaMemcpyDeviceToHost, ctx->stream));
  GBEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  const unsigned long long* h = ctx->h_stats;
  if (stats) {
    stats->pairs_total = pairs_total;
    stats->pairs_coplanar = (int64_t)h[ST_COP];
    stats->pairs_parallel = (int64_t)h[ST_PAR];
    stats->pairs_orthogonal = (int64_t)h[ST_ORTH];
    stats->pairs_far = (int64_t)h[ST_FAR];
    stats->not_converged = (int64_t)h[ST_NONCONV];
    stats->nonfinite = (int64_t)h[ST_NONFINITE];
    stats->near_evals = (int64_t)h[ST_NEAR_EVALS];
    stats->far_evals = (int64_t)h[ST_FAR_EVALS];
    double f;
    memcpy(&f, &h[ST_FAR_FLOPS], sizeof(double));
    stats->far_flops = f;
    stats->pairs_near_romberg = (int64_t)h[ST_ROMB];
    for (int b = 0; b < 4; ++b) stats->pairs_near_band[b] = b < kNearBands ? (int64_t)h[ST_BAND0 + b] : 0;
  }
  if (h[ST_NONFINITE]) {
    unsigned long long b = h[ST_FIRST_BAD];
    return ctx->fail(GBEM_ENUMERIC, "non-finite integrand sample (pair " +
                                        std::to_string(b >> 32) + "," +
                                        std::to_string(b & 0xffffffffull) + ")");
  }
  return GBEM_OK;
}

}  // namespace

int gbem_internal_init_tables(gbem_ctx* ctx) {
  double gx[kQMax + 1][kQMax], gw[kQMax + 1][kQMax];
  legendre_table(gx, gw);
  GBEM_CUDA(ctx, cudaMemcpyToSymbol(c_gx, gx, sizeof(gx)));
  GBEM_CUDA(ctx, cudaMemcpyToSymbol(c_gw, gw, sizeof(gw)));
  double nx[kNearBands][48] = {}, nw[kNearBands][48] = {};
  for (int b = 0; b < kNearBands; ++b) legendre_nodes(near_nodes(b), nx[b], nw[b]);
  GBEM_CUDA(ctx, cudaMemcpyToSymbol(c_nx, nx, sizeof(nx)));
  GBEM_CUDA(ctx, cudaMemcpyToSymbol(c_nw, nw, sizeof(nw)));
  {
    double kr[kQMax + 1][kQMax] = {}, kp[kQMax + 1][kQMax] = {};
    static double kpp[kQProd + 1][kQProd + 1][kQProd * kQProd];
    for (int q = 1; q <= kQMax; ++q)
      for (int k = 0; k < q; ++k) {
        const double t = gw[q][k] * (1.0 + gx[q][k]);
        kr[q][k] = 1.0 / (t * t);
        kp[q][k] = 1.0 / (gw[q][k] * gw[q][k]);
      }
    for (int q1 = 1; q1 <= kQProd; ++q1)
      for (int q2 = 1; q2 <= kQProd; ++q2)
        for (int a = 0; a < q1; ++a)
          for (int b = 0; b < q2; ++b) {
            const double t = gw[q1][a] * gw[q2][b];
            kpp[q1][q2][a * q2 + b] = 1.0 / (t * t);
          }
    GBEM_CUDA(ctx, cudaMemcpyToSymbol(c_kr, kr, sizeof(kr)));
    GBEM_CUDA(ctx, cudaMemcpyToSymbol(c_kp, kp, sizeof(kp)));
    GBEM_CUDA(ctx, cudaMemcpyToSymbol(c_kpp, kpp, sizeof(kpp)));
  }
  int8_t fast[512];
  for (int k = 0; k < 512; ++k) fast[k] = -1;
  if (!getenv("GBEM_NO_FAST_FAR")) {  // experiments: every far pair through the generic kernels
#define GBEM_FAST_ENTRY(D, TYPE, Q1, Q2) \
  static_assert(D < kFastMax, "descriptor index"); \
  fast[(int)TYPE | (Q1 - 1) << 2 | Q2 << 5] = D;
    GBEM_FAST_DESCS(GBEM_FAST_ENTRY)
#undef GBEM_FAST_ENTRY
  }
  GBEM_CUDA(ctx, cudaMemcpyToSymbol(c_fast_idx, fast, sizeof(fast)));
  return GBEM_OK;
}

int gbem_internal_upload_panels(gbem_ctx* ctx, const gbem_panels* P, int64_t n, bool device_ptrs) {
  if (n < 0 || n >= (1 << 24)) return ctx->fail(GBEM_EINVAL, "panel count out of range");
  if (n == 0) return GBEM_OK;
  if (!P || !P->axis || !P->level || !P->a_lo || !P->a_hi || !P->b_lo || !P->b_hi)
    return ctx->fail(GBEM_EINVAL, "null panel array");
  int rc = grow(ctx, (void**)&ctx->d_panels, sizeof(DPanel) * (size_t)n, &ctx->panel_cap, sizeof(DPanel));
  if (rc) return rc;
  if (device_ptrs) {
    k_pack_panels<<<(int)((n + 255) / 256), 256, 0, ctx->stream>>>(P->axis, P->level, P->a_lo, P->a_hi,
                                                                   P->b_lo, P->b_hi, (int)n, ctx->d_panels);
    GBEM_LAUNCH_CHECK(ctx);
    return GBEM_OK;
  }
  std::vector<DPanel> h((size_t)n);
  for (int64_t k = 0; k < n; ++k) {
    if (P->axis[k] > 2) return ctx->fail(GBEM_EINVAL, "panel axis must be 0, 1 or 2");
    if (!(P->a_lo[k] < P->a_hi[k]) || !(P->b_lo[k] < P->b_hi[k]))
      return ctx->fail(GBEM_EINVAL, "panel spans must satisfy lo < hi (panel " + std::to_string(k) + ")");
    DPanel d;
    d.level = P->level[k];
    d.a0 = P->a_lo[k];
    d.a1 = P->a_hi[k];
    d.b0 = P->b_lo[k];
    d.b1 = P->b_hi[k];
    d.axis = P->axis[k];
    d.pad = 0;
    h[(size_t)k] = d;
  }
  GBEM_CUDA(ctx, cudaMemcpyAsync(ctx->d_panels, h.data(), sizeof(DPanel) * (size_t)n,
                                 cudaMemcpyHostToDevice, ctx->stream));
  GBEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));  // h is a stack vector
  return GBEM_OK;
}

// Assemble rows [row_begin, row_end) of the upper triangle into ctx->d_A.
int gbem_internal_assemble(gbem_ctx* ctx, int64_t n, int64_t row_begin, int64_t row_end,
                           const gbem_quad_config* cfg_in, gbem_assembly_stats* stats, bool symmetrize,
                           double* out, int64_t ld_out, bool full_rows, bool out_col_major) {
  gbem_quad_config cfg;
  int rc = prepare_work(ctx, cfg_in, &cfg);
  if (rc) return rc;
  if (stats) *stats = gbem_assembly_stats{};
  if (n == 0) return GBEM_OK;
  const int nbt = (int)((n + kTile - 1) / kTile);
  const int bi0 = (int)(row_begin / kTile), bi1 = (int)((row_end - 1) / kTile);
  const int nrows_t = bi1 - bi0 + 1;
  std::vector<long long> rowoff((size_t)nrows_t + 1);
  long long total_tiles = 0;
  for (int r = 0; r < nrows_t; ++r) {
    rowoff[(size_t)r] = total_tiles;
    total_tiles += full_rows ? nbt : nbt - (bi0 + r);
  }
  rowoff[(size_t)nrows_t] = total_tiles;
  // queue capacity: 2^27 entries (1 GiB) or what the problem needs
  long long need = std::min<long long>(total_tiles * kTile * kTile, 1ll << 27);
  // test hook: a small queue splits a small problem into many chunks (tests/test_gpu_assembly.py)
  if (const char* e = getenv("GBEM_QUEUE_CAP")) need = std::min<long long>(need, std::max<long long>(kTile * kTile, atoll(e)));
  rc = grow(ctx, (void**)&ctx->d_queue, sizeof(uint64_t) * (size_t)need, &ctx->queue_cap, sizeof(uint64_t));
  if (rc) return rc;
  rc = grow(ctx, (void**)&ctx->d_plan, sizeof(uint32_t) * (size_t)ctx->queue_cap, &ctx->plan_cap, sizeof(uint32_t));
  if (rc) return rc;
  rc = grow(ctx, (void**)&ctx->d_kp, sizeof(uint64_t) * (size_t)ctx->queue_cap, &ctx->kp_cap, sizeof(uint64_t));
  if (rc) return rc;
  rc = prepare_cinfo(ctx, n);
  if (rc) return rc;
  long long* d_rowoff = nullptr;
  GBEM_CUDA(ctx, cudaMallocAsync(&d_rowoff, sizeof(long long) * rowoff.size(), ctx->stream));
  GBEM_CUDA(ctx, cudaMemcpyAsync(d_rowoff, rowoff.data(), sizeof(long long) * rowoff.size(),
                                 cudaMemcpyHostToDevice, ctx->stream));
  // destination: the context matrix (entry (i, j >= i) at A[i*lda + j]) or a
  // caller row block, row-major (entry at out[(i - row_begin)*ld_out + j]) or
  // column-major (out[j*ld_out + i - row_begin], the sharded solve's layout)
  OutSpec o{ctx->d_A, (long long)ctx->lda, 1, nullptr, nullptr};
  if (out && !out_col_major) {
    o.A = out - row_begin * ld_out;
    o.lda = (long long)ld_out;
  } else if (out) {
    o.A = out - row_begin;
    o.lda = 1;
    o.ldc = (long long)ld_out;
  }
  const long long tiles_per_chunk =
      std::max<long long>(1, (getenv("GBEM_QUEUE_CAP") ? need : (long long)ctx->queue_cap) / (kTile * kTile));
  float ms_cls = 0, ms_far = 0, ms_near = 0;
  bool timing = stats != nullptr;
  static const bool defer_romberg = getenv("GBEM_NO_ROMBERG_DEFER") == nullptr;
  if (defer_romberg) {
    if (!ctx->d_romb) {
      GBEM_CUDA(ctx, cudaMalloc(&ctx->d_romb, sizeof(uint64_t) * kRombCap));
      GBEM_CUDA(ctx, cudaMalloc(&ctx->d_romb_cnt, sizeof(uint32_t) * 2));
    }
    GBEM_CUDA(ctx, cudaMemsetAsync(ctx->d_romb_cnt, 0, sizeof(uint32_t) * 2, ctx->stream));
  }
  // Classification of chunk t + 1 runs on its own stream, into a second queue / plan / offsets set,
  // while chunk t is evaluated: the classifier is integer / FP32 issue-bound, the far field FP64-pipe
  // bound, and its CTAs fit beside the far-field kernels' as those drain.  Per-phase timing
  // (stats) keeps the phases one after the other.
  static const bool pipeline_env = getenv("GBEM_NO_CLASSIFY_PIPELINE") == nullptr;
  const long long nchunks = (total_tiles + tiles_per_chunk - 1) / tiles_per_chunk;
  const bool pipelined = !timing && pipeline_env && nchunks >= 2;
  uint64_t* qbuf[2] = {ctx->d_queue, ctx->d_queue};
  uint32_t* pbuf[2] = {ctx->d_plan, ctx->d_plan};
  uint32_t* obuf[2] = {ctx->d_offsets, ctx->d_offsets};
  cudaStream_t cs = ctx->stream;
  if (pipelined) {
    rc = grow(ctx, (void**)&ctx->d_queue2, sizeof(uint64_t) * (size_t)ctx->queue_cap, &ctx->queue2_cap, sizeof(uint64_t));
    if (rc) return rc;
    rc = grow(ctx, (void**)&ctx->d_plan2, sizeof(uint32_t) * (size_t)ctx->queue_cap, &ctx->plan2_cap, sizeof(uint32_t));
    if (rc) return rc;
    if (!ctx->d_offsets2) GBEM_CUDA(ctx, cudaMalloc(&ctx->d_offsets2, sizeof(uint32_t) * (kNumKeys + 1)));
    if (!ctx->cls_stream) {
      GBEM_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->cls_stream, cudaStreamNonBlocking));
      for (cudaEvent_t& e : ctx->ev_cls) GBEM_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    qbuf[1] = ctx->d_queue2;
    pbuf[1] = ctx->d_plan2;
    obuf[1] = ctx->d_offsets2;
    cs = ctx->cls_stream;
    GBEM_CUDA(ctx, cudaEventRecord(ctx->ev_cls[0], ctx->stream));
    GBEM_CUDA(ctx, cudaStreamWaitEvent(cs, ctx->ev_cls[0], 0));
  }
  cudaEventRecord(ctx->ev[0], ctx->stream);
  long long chunk = 0;
  for (long long t0 = 0; t0 < total_tiles; t0 += tiles_per_chunk, ++chunk) {
    long long nt = std::min(tiles_per_chunk, total_tiles - t0);
    const int b = pipelined ? (int)(chunk & 1) : 0;
    if (pipelined && chunk >= 2)  // the evaluation of chunk - 2 has finished with this buffer set
      GBEM_CUDA(ctx, cudaStreamWaitEvent(cs, ctx->ev_cls[3 + b], 0));
    cudaEventRecord(ctx->ev[5], cs);
    GBEM_CUDA(ctx, cudaMemsetAsync(ctx->d_counts, 0, sizeof(uint32_t) * kNumKeys, cs));
    k_classify<false><<<(unsigned)nt, kClassifyThreads, 0, cs>>>(
        (const CPanel*)ctx->d_cinfo, (int)n, (int)row_begin, (int)row_end, bi0, nbt, d_rowoff, nrows_t, t0,
        cfg.near_ratio, ctx->d_counts, ctx->d_cursors, qbuf[b], pbuf[b], ctx->d_kp, full_rows ? 1 : 0);
    GBEM_LAUNCH_CHECK(ctx);
    k_scan<<<1, 1024, 0, cs>>>(ctx->d_counts, obuf[b], ctx->d_cursors, ctx->d_stats);
    GBEM_LAUNCH_CHECK(ctx);
    k_classify<true><<<(unsigned)nt, kClassifyThreads, 0, cs>>>(
        (const CPanel*)ctx->d_cinfo, (int)n, (int)row_begin, (int)row_end, bi0, nbt, d_rowoff, nrows_t, t0,
        cfg.near_ratio, ctx->d_counts, ctx->d_cursors, qbuf[b], pbuf[b], ctx->d_kp, full_rows ? 1 : 0);
    GBEM_LAUNCH_CHECK(ctx);
    cudaEventRecord(ctx->ev[6], cs);
    if (timing) {
      GBEM_CUDA(ctx, cudaEventSynchronize(ctx->ev[6]));
      float a = 0;
      cudaEventElapsedTime(&a, ctx->ev[5], ctx->ev[6]);
      ms_cls += a;
    }
    if (pipelined) {
      GBEM_CUDA(ctx, cudaEventRecord(ctx->ev_cls[1 + b], cs));
      GBEM_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_cls[1 + b], 0));
    }
    // the evaluation kernels take their queue from the context: point it at this chunk's set
    ctx->d_queue = qbuf[b];
    ctx->d_plan = pbuf[b];
    ctx->d_offsets = obuf[b];
    rc = run_eval(ctx, o, cfg, timing ? &ms_far : nullptr, timing ? &ms_near : nullptr, defer_romberg);
    ctx->d_queue = qbuf[0];
    ctx->d_plan = pbuf[0];
    ctx->d_offsets = obuf[0];
    if (rc) return rc;
    if (pipelined) GBEM_CUDA(ctx, cudaEventRecord(ctx->ev_cls[3 + b], ctx->stream));
  }
  if (defer_romberg) {  // the near-contact pairs of every chunk, one warp each
    cudaEventRecord(ctx->ev[2], ctx->stream);
    k_near_warp<<<ctx->num_sms * 8, 128, 0, ctx->stream>>>(ctx->d_panels, ctx->d_romb, ctx->d_offsets, o, cfg.rel_tol,
                                                          cfg.max_levels, ctx->d_stats, nullptr, ctx->d_romb_cnt);
    GBEM_LAUNCH_CHECK(ctx);
    cudaEventRecord(ctx->ev[3], ctx->stream);
    if (timing) {
      GBEM_CUDA(ctx, cudaEventSynchronize(ctx->ev[3]));
      float a = 0;
      cudaEventElapsedTime(&a, ctx->ev[2], ctx->ev[3]);
      ms_near += a;
    }
  }
  if (symmetrize) {
    const int snbt = (int)((n + kSymTile - 1) / kSymTile);
    long long ntiles = (long long)snbt * (snbt + 1) / 2;
    k_symmetrize<<<(unsigned)ntiles, 256, 0, ctx->stream>>>(ctx->d_A, (long long)ctx->lda, (int)n, snbt);
    GBEM_LAUNCH_CHECK(ctx);
  }
  cudaEventRecord(ctx->ev[1], ctx->stream);
  GBEM_CUDA(ctx, cudaFreeAsync(d_rowoff, ctx->stream));
  long long pairs = 0;
  for (int64_t i = row_begin; i < row_end; ++i) pairs += full_rows ? n : n - i;
  if (stats) {
    rc = finish_stats(ctx, stats, pairs);
    float tot = 0;
    cudaEventElapsedTime(&tot, ctx->ev[0], ctx->ev[1]);
    stats->ms_classify = ms_cls;
    stats->ms_far = ms_far;
    stats->ms_near = ms_near;
    stats->ms_total = tot;
    return rc;
  }
  if (ctx->async) {  // non-finite check deferred to gbem_ctx_sync
    GBEM_CUDA(ctx, cudaMemcpyAsync(ctx->h_stats, ctx->d_stats, sizeof(unsigned long long) * ST_COUNT,
                                   cudaMemcpyDeviceToHost, ctx->stream));
    ctx->stats_pending = true;
    return GBEM_OK;
  }
  return finish_stats(ctx, nullptr, pairs);
}

int gbem_internal_check_pending_stats(gbem_ctx* ctx) {
  if (!ctx->stats_pending) return GBEM_OK;
  ctx->stats_pending = false;
  const unsigned long long* h = ctx->h_stats;
  if (h[ST_NONFINITE]) {
    unsigned long long b = h[ST_FIRST_BAD];
    return ctx->fail(GBEM_ENUMERIC, "non-finite integrand sample (pair " + std::to_string(b >> 32) + "," +
                                        std::to_string(b & 0xffffffffull) + ")");
  }
  return GBEM_OK;
}

int gbem_internal_pair_list(gbem_ctx* ctx, int64_t npairs, const gbem_quad_config* cfg_in,
                            double* d_out, int32_t* d_conv, gbem_assembly_stats* stats) {
  gbem_quad_config cfg;
  int rc = prepare_work(ctx, cfg_in, &cfg);
  if (rc) return rc;
  if (npairs == 0) return GBEM_OK;
  if (npairs > (1 << 23)) return ctx->fail(GBEM_EINVAL, "at most 2^23 pairs per call");
  rc = grow(ctx, (void**)&ctx->d_queue, sizeof(uint64_t) * (size_t)npairs, &ctx->queue_cap, sizeof(uint64_t));
  if (rc) return rc;
  rc = grow(ctx, (void**)&ctx->d_plan, sizeof(uint32_t) * (size_t)ctx->queue_cap, &ctx->plan_cap, sizeof(uint32_t));
  if (rc) return rc;
  rc = prepare_cinfo(ctx, 2 * npairs);
  if (rc) return rc;
  GBEM_CUDA(ctx, cudaMemsetAsync(ctx->d_counts, 0, sizeof(uint32_t) * kNumKeys, ctx->stream));
  int blocks = (int)((npairs + 255) / 256);
  k_classify_list<false><<<blocks, 256, 0, ctx->stream>>>((const CPanel*)ctx->d_cinfo, (int)npairs, cfg.near_ratio,
                                                          ctx->d_counts, ctx->d_cursors, ctx->d_queue,
                                                          ctx->d_plan);
  GBEM_LAUNCH_CHECK(ctx);
  k_scan<<<1, 1024, 0, ctx->stream>>>(ctx->d_counts, ctx->d_offsets, ctx->d_cursors, ctx->d_stats);
  GBEM_LAUNCH_CHECK(ctx);
  k_classify_list<true><<<blocks, 256, 0, ctx->stream>>>((const CPanel*)ctx->d_cinfo, (int)npairs, cfg.near_ratio,
                                                         ctx->d_counts, ctx->d_cursors, ctx->d_queue,
                                                         ctx->d_plan);
  GBEM_LAUNCH_CHECK(ctx);
  OutSpec o{nullptr, 0, 0, d_out, d_conv};
  rc = run_eval(ctx, o, cfg, nullptr, nullptr);
  if (rc) return rc;
  return finish_stats(ctx, stats, npairs);
}

namespace {
// Q (rows x K, row-major, ldq) = Ablk (rows x n, row i contiguous, ld) * P (n x K,
// row-major: one row of K values per panel, ldp).  32 rows per CTA (4 per warp);
// P is staged through shared memory in 256-panel chunks, KC right-hand sides per
// pass.  HBM-bound on Ablk (8 B per entry per pass) for K <= KC.
template <int KC, int RW>
__global__ void __launch_bounds__(256, 2)
    k_rowblock_matvec(const double* __restrict__ Ab, long long ld, int rows, int n, const double* __restrict__ P,
                      long long ldp, int K, int q0, double* __restrict__ Q, long long ldq) {
  __shared__ double ps[KC * 256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = blockIdx.x * (8 * RW) + warp * RW;
  const int kc = min(KC, K - q0);
  double acc[RW][KC];
#pragma unroll
  for (int u = 0; u < RW; ++u)
#pragma unroll
    for (int q = 0; q < KC; ++q) acc[u][q] = 0.0;
  for (int j0 = 0; j0 < n; j0 += 256) {
    const int jn = min(256, n - j0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < 256 * KC; idx += blockDim.x) {
      const int jj = idx / KC, q = idx % KC;
      ps[q * 256 + jj] = (jj < jn && q < kc) ? P[(long long)(j0 + jj) * ldp + q0 + q] : 0.0;
    }
    __syncthreads();
#pragma unroll 2
    for (int t = 0; t < 8; ++t) {
      const int c = lane + 32 * t;
      double pv[KC];
#pragma unroll
      for (int q = 0; q < KC; ++q) pv[q] = ps[q * 256 + c];  // one shared load per P value, reused RW times
      double av[RW];
#pragma unroll
      for (int u = 0; u < RW; ++u) av[u] = (c < jn && r0 + u < rows) ? __ldcs(Ab + (long long)(r0 + u) * ld + j0 + c) : 0.0;
#pragma unroll
      for (int u = 0; u < RW; ++u)
#pragma unroll
        for (int q = 0; q < KC; ++q) acc[u][q] = fma(av[u], pv[q], acc[u][q]);
    }
  }
#pragma unroll
  for (int u = 0; u < RW; ++u) {
    const int r = r0 + u;
#pragma unroll
    for (int q = 0; q < KC; ++q) {
      double v = acc[u][q];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0 && r < rows && q < kc) Q[(long long)r * ldq + q0 + q] = v;
    }
  }
}
}  // namespace

namespace {
// Wide right-hand sides (K > 8): the same product on the FP64 tensor cores.
// CTA = 64 rows x FN*8 columns of Q, 4 warps of 16 rows (2 x FN DMMA m8n8k4
// fragments each), n consumed in 16-wide slabs through a 2-stage cp.async
// pipeline (A rows 128 B contiguous, P slab rows K*8 B contiguous).
template <int FN>
__global__ void __launch_bounds__(128)
    k_rowblock_mm(const double* __restrict__ Ab, long long ld, int rows, int n, const double* __restrict__ P,
                  long long ldp, int K, int q0, double* __restrict__ Q, long long ldq, int vec16) {
  constexpr int TM = 64, KS = 16, NW = FN * 8;
  constexpr int LA = KS + 4, LP = NW + 4;  // padded smem strides (doubles)
  __shared__ __align__(16) double As[2][TM * LA];
  __shared__ __align__(16) double Ps[2][KS * LP];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int r0 = blockIdx.x * TM;
  const int ncols = min(NW, K - q0);
  auto load = [&](int s, int buf) {
    const int k0 = s * KS;
    for (int c = tid; c < TM * KS / 2; c += 128) {  // A: 64 rows x KS/2 double2
      const int r = c / (KS / 2), kk = (c % (KS / 2)) * 2;
      const int gr = r0 + r, gk = k0 + kk;
      if (vec16) {
        int bytes = 0;
        const double* src = Ab;
        if (gr < rows && gk < n) {
          bytes = gk + 1 < n ? 16 : 8;
          src = Ab + (long long)gr * ld + gk;
        }
        gbem_gemm::cp_async16(&As[buf][r * LA + kk], src, bytes);
      } else {  // unaligned leading dimensions: element-wise 8-byte copies
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const bool ok = gr < rows && gk + e < n;
          gbem_gemm::cp_async8(&As[buf][r * LA + kk + e], ok ? Ab + (long long)gr * ld + gk + e : Ab, ok ? 8 : 0);
        }
      }
    }
    for (int c = tid; c < KS * NW / 2; c += 128) {  // P: KS rows x NW/2 double2
      const int kk = c / (NW / 2), q = (c % (NW / 2)) * 2;
      const int gk = k0 + kk;
      if (vec16) {
        int bytes = 0;
        const double* src = P;
        if (gk < n && q < ncols) {
          bytes = q + 1 < ncols ? 16 : 8;
          src = P + (long long)gk * ldp + q0 + q;
        }
        gbem_gemm::cp_async16(&Ps[buf][kk * LP + q], src, bytes);
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const bool ok = gk < n && q + e < ncols;
          gbem_gemm::cp_async8(&Ps[buf][kk * LP + q + e], ok ? P + (long long)gk * ldp + q0 + q + e : P, ok ? 8 : 0);
        }
      }
    }
  };
  double acc[2][FN][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int S = (n + KS - 1) / KS;
  load(0, 0);
  gbem_gemm::cp_async_commit();
  for (int s = 0; s < S; ++s) {
    if (s + 1 < S) load(s + 1, (s + 1) & 1);
    gbem_gemm::cp_async_commit();
    gbem_gemm::cp_async_wait<1>();
    __syncthreads();
    const double* as = &As[s & 1][(warp * 16 + g) * LA + t4];
    const double* ps = &Ps[s & 1][t4 * LP + g];
#pragma unroll
    for (int kk = 0; kk < KS; kk += 4) {
      const double a0 = as[kk], a1 = as[8 * LA + kk];
#pragma unroll
      for (int j = 0; j < FN; ++j) {
        const double b = ps[kk * LP + j * 8];
        gbem_gemm::dmma(acc[0][j][0], acc[0][j][1], a0, b);
        gbem_gemm::dmma(acc[1][j][0], acc[1][j][1], a1, b);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = r0 + warp * 16 + i * 8 + g;
    if (r >= rows) continue;
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int q = j * 8 + 2 * t4 + e;
        if (q < ncols) Q[(long long)r * ldq + q0 + q] = acc[i][j][e];
      }
  }
}
}  // namespace

int gbem_internal_rowblock_matvec(gbem_ctx* ctx, const double* Ab, int64_t ld, int64_t rows, int64_t n,
                                  const double* P, int64_t ldp, int64_t K, double* Q, int64_t ldq) {
  if (rows <= 0 || K <= 0) return GBEM_OK;
  if (K <= 8) {  // HBM-bound: one pass of the FP64-pipe kernel
    k_rowblock_matvec<8, 4><<<(unsigned)((rows + 31) / 32), 256, 0, ctx->stream>>>(Ab, ld, (int)rows, (int)n, P,
                                                                                 ldp, (int)K, 0, Q, ldq);
    GBEM_LAUNCH_CHECK(ctx);
    return GBEM_OK;
  }
  // DMMA: up to 64 right-hand sides per pass (intensity K/4 flop/B: tensor-bound above K ~ 20)
  const int vec16 = ((ld | ldp) % 2 == 0 && ((uintptr_t)Ab % 16) == 0 && ((uintptr_t)P % 16) == 0) ? 1 : 0;
  for (int q0 = 0; q0 < K; q0 += 64) {
    const int w = (int)std::min<int64_t>(64, K - q0);
    const unsigned grid = (unsigned)((rows + 63) / 64);
    if (w <= 16)
      k_rowblock_mm<2><<<grid, 128, 0, ctx->stream>>>(Ab, ld, (int)rows, (int)n, P, ldp, (int)K, q0, Q, ldq,
                                                         vec16);
    else if (w <= 32)
      k_rowblock_mm<4><<<grid, 128, 0, ctx->stream>>>(Ab, ld, (int)rows, (int)n, P, ldp, (int)K, q0, Q, ldq,
                                                         vec16);
    else
      k_rowblock_mm<8><<<grid, 128, 0, ctx->stream>>>(Ab, ld, (int)rows, (int)n, P, ldp, (int)K, q0, Q, ldq,
                                                         vec16);
    GBEM_LAUNCH_CHECK(ctx);
  }
  return GBEM_OK;
}

// gbem_solver.cu — dense SPD solve on B200: blocked right-looking Cholesky with
// an FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) trailing update, K-RHS
// triangular solves, residual recomputed from the original matrix.
//
// Replaces cholesky_solve + residual_norm (proj/include/gbem/solver.hpp:17-50).
// Same contract: SPD input, "matrix not positive definite (pivot at row k)" on a
// non-positive pivot (solver.hpp:31-33), relative residual ||Ax-b||/||b||
// recomputed from the unfactored matrix (solver.hpp:47).
//
// Storage: column-major A (lda), lower triangle overwritten by L; the strict
// upper triangle is left untouched and the original diagonal is saved, so the
// residual uses the original A.  Block size NB = 128:
//   k_potrf_diag  : one CTA factors the NB x NB diagonal block in shared memory
//                   and forms inv(L11) (kept for the solves);
//   k_trsm_rows   : L21 = A21 * inv(L11)^T (trsm as a DMMA GEMM on 32-row strips, in place);
//   k_syrk_gen    : A22 -= L21 * L21^T on lower 64x64 tiles (the O(n^3) part).
// Bordered mode (ctx->border > 0, the K-RHS extraction): the K rows below the
// matrix hold B^T and ride along as extra rows of every trsm and update, so the
// factorisation also leaves Y = inv(L) B (forward substitution) and -B^T A^-1 B.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "gbem_ctx.cuh"
#include "gbem_common.cuh"
#include "gbem_dmma_gemm.cuh"
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace {

using namespace gbem_gemm;
constexpr int NB = 128;       // Cholesky block size (diagonal blocks, trailing-update K)
// trailing update: 64 x 64 tiles, 2 x 2 warps, double-buffered slabs, 4 CTAs per
// SM (tools/gemm_bench.cu: 28.0 TFLOP/s at K = 128 vs 25.6 for 128 x 64 tiles)
using UpdShape = GenShape<64, 64, 2, 2, 2>;
#define kUpdate k_syrk_gen<64, 64, 2, 2, 2, 4>
// shared memory of an update CTA padded so that only 3 fit on an SM (4 x 61 KB >
// 228 KB) and a trsm or band CTA (<= 38 KB, <= 16K registers) fits beside them
constexpr size_t kUpdSmemPadded = 60 * 1024;
static_assert(UpdShape::SMEM <= kUpdSmemPadded, "padding");
// The same update with its operand slabs staged by bulk copies (TMA engine, mbarrier pipeline;
// gbem_dmma_gemm.cuh): 35.9 vs 34.3 TFLOP/s at K = 1,536, bit-identical results.  It needs
// K % 16 == 0 and 16-byte copies, so ragged panels take the cp.async kernel.
using BulkUpd = BulkShape<16, 3>;
#define kUpdateBulk k_syrk_bulk<16, 3, 4, true>
static_assert(BulkUpd::SMEM <= kUpdSmemPadded, "padding");

inline void launch_update(gbem_ctx* ctx, dim3 grid, bool padded, cudaStream_t st, double* C, long long ldc,
                          const double* A, long long lda, int M, int K, int split, int band,
                          unsigned* band_done = nullptr) {
  static const bool use_bulk = getenv("GBEM_UPDATE_CPASYNC") == nullptr;
  // an odd row count is copied rounded up to 16 bytes: the next element must lie inside the column
  const long long row0 = (A - ctx->d_A) % lda;
  const bool bulk = use_bulk && K % 16 == 0 && lda % 2 == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0 &&
                    ((M & 1) == 0 || row0 + M < lda);
  if (bulk)
    kUpdateBulk<<<grid, BulkUpd::THREADS, padded ? kUpdSmemPadded : BulkUpd::SMEM, st>>>(C, ldc, A, lda, M, K, split,
                                                                                         band, band_done);
  else
    kUpdate<<<grid, UpdShape::THREADS, padded ? kUpdSmemPadded : UpdShape::SMEM, st>>>(C, ldc, A, lda, M, K, split,
                                                                                       band, band_done);
}
// Factor the kb x kb (kb <= NB = 128) diagonal block and invert its factor, in
// shared memory, by 32-column panels:
//   1. warp 0 factors the 32 x 32 diagonal sub-block in registers (lane i owns
//      row i; pivots and column entries move by __shfl_sync, no block barriers)
//      and inverts it the same way;
//   2. all warps form the panel rows below: L_rp = A_rp * inv(L_pp)^T;
//   3. all warps apply the rank-32 update to the trailing sub-block (4 x 4
//      register tiles);
// then the off-diagonal 32 x 32 blocks of X = inv(L) follow from
// X_rp = -X_rr * sum_{q=p}^{r-1} L_rq X_qp.  L goes back to A (lower), X to Linv
// (column-major, ld = NB) for the GEMM-form trsm and the triangular solves.
// X(r,c), r > c, is kept at a[r*LD + c] (the strict upper half), its diagonal
// in xd.  info[0] receives the first failing global row (atomicMin); a failed
// pivot continues as 1 so the launch sequence stays fixed.
#ifdef GBEM_POTRF_TIMING
__device__ long long g_potrf_clk[128];
#define POTRF_TICK(k) \
  if (threadIdx.x == 0) g_potrf_clk[k] = clock64();
#define POTRF_TICK_T(k, t) \
  if (threadIdx.x == (t)) g_potrf_clk[k] = clock64();
#else
#define POTRF_TICK(k)
#define POTRF_TICK_T(k, t)
#endif
constexpr int kPotrfThreads = 512;
constexpr int kPotrfWarps = kPotrfThreads / 32;
constexpr int kPanel = 32;
constexpr int kInvSlots = 6;  // sums T_rp, p < r <= 3
constexpr size_t kPotrfSmem = (size_t)(NB * (NB + 1) + NB + kInvSlots * kPanel * (kPanel + 1)) * sizeof(double);

// Off-diagonal 32 x 32 blocks of X = inv(L) of the diagonal block:
// X_rp = -X_rr * T_rp, T_rp = sum_{q=p}^{r-1} L_rq X_qp, for p < r.  X(r,c), r > c,
// lives in the strict upper half a[r*LD + c], its diagonal in xd; T_rp
// accumulates in tmp[r(r-1)/2 + p][32][33].  Part 1: one product L_rq X_qp
// (32 x 32 x 32, strided 4 x 4 register tiles on a two-warp team, gt = index
// 0..63 in the team) -- all products with the same q run while warp 0 factors
// panel q + 1 (L_rq and X_qp are final by then), on the warps off warp 0's
// sub-partition.  Part 2 applies -X_rr beside the panel-row step of panel r
// (disjoint rows of the same columns).
__device__ __forceinline__ int inv_slot(int r, int p) { return r * (r - 1) / 2 + p; }
__device__ __forceinline__ void potrf_inv_part1(const double* a, const double* xd, double* tmp, int r, int p,
                                                int q, int gt) {
  constexpr int LD = NB + 1, TLD = kPanel + 1;
  const int R0 = r * kPanel, tx = gt & 7, ty = gt >> 3;
  double acc[4][4] = {};
#pragma unroll 4
  for (int m = q * kPanel; m < (q + 1) * kPanel; ++m) {
    double lr[4], xc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) lr[u] = a[m * LD + R0 + ty + 8 * u];  // L(R0+i, m)
    const double dg = xd[m];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int c = p * kPanel + tx + 8 * v;
      const double up = a[m * LD + c];
      xc[v] = m > c ? up : 0.0;
      xc[v] = m == c ? dg : xc[v];  // X(m, c)
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] = fma(lr[u], xc[v], acc[u][v]);
  }
  double* t = tmp + inv_slot(r, p) * kPanel * TLD;
  const bool first = q == p;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      double& d = t[(ty + 8 * u) * TLD + tx + 8 * v];
      d = first ? acc[u][v] : d + acc[u][v];
    }
}

// rows ty + 8 (u0 + u), u < NU, of X_rp (a team of 64 threads per NU = 4 block,
// two teams per block with NU = 2); X_rr is lower triangular, so the m-loop
// stops at the last row of the slice
template <int NU>
__device__ __forceinline__ void potrf_inv_part2(double* a, const double* xd, const double* tmp, int rbk, int pb,
                                                int tx, int ty, int u0) {
  constexpr int LD = NB + 1, TLD = kPanel + 1;
  const int R0 = rbk * kPanel, mend = 8 * (u0 + NU);
  double acc[NU][4] = {};
#pragma unroll 4
  for (int m = 0; m < mend; ++m) {
    double xr[NU], tv[4];
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const int i = ty + 8 * (u0 + u);
      const double up = a[(R0 + i) * LD + R0 + m], dg = xd[R0 + i];
      xr[u] = m < i ? up : 0.0;
      xr[u] = m == i ? dg : xr[u];  // X(R0+i, R0+m)
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) tv[v] = tmp[inv_slot(rbk, pb) * kPanel * TLD + m * TLD + tx + 8 * v];
#pragma unroll
    for (int u = 0; u < NU; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] = fma(xr[u], tv[v], acc[u][v]);
  }
#pragma unroll
  for (int u = 0; u < NU; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v)
      a[(R0 + ty + 8 * (u0 + u)) * LD + pb * kPanel + tx + 8 * v] = -acc[u][v];  // X(R0+i, col)
}

__global__ void __launch_bounds__(kPotrfThreads)
    k_potrf_diag(double* A, long long lda, int kb, int row0, double* Linv, int* info,
                 const unsigned* wait_ctr = nullptr, unsigned wait_target = 0) {
  extern __shared__ __align__(16) double sm[];
  constexpr int LD = NB + 1;
  double* a = sm;              // [NB][LD] column-major: a[c*LD + r]
  double* xd = a + NB * LD;    // diag of X (= 1 / diag of L)
  double* tmp = xd + NB;       // [3][32][33] products of the X assembly
  const int tid = threadIdx.x, lane = tid & 31;
  // warp index through a shuffle: ptxas then knows it is warp-uniform, and the
  // shuffles inside `if (warp == 0)` compile without divergence handling
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  POTRF_TICK(23);
  // launched ahead of its producer (the band tiles of a combined update,
  // k_syrk_gen band < 0): wait until they have all stored
  if (wait_ctr) {
    if (tid == 0) {
      unsigned v;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(wait_ctr) : "memory");
        if (v >= wait_target) break;
        __nanosleep(64);
      }
      __threadfence();
    }
    __syncthreads();
  }
  // load the block (L2 loads: the block may have been written during this kernel): 8 independent global loads in flight per thread per batch
  for (int idx0 = tid; idx0 < NB * NB; idx0 += 8 * kPotrfThreads) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = idx0 + u * kPotrfThreads, c = idx / NB, r = idx % NB;
      v[u] = 0.0;
      if (idx < NB * NB) {
        if (r < kb && c < kb) v[u] = r >= c ? __ldcg(A + (long long)c * lda + r) : 0.0;
        else if (r == c) v[u] = 1.0;  // pad the ragged last block with the identity
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int idx = idx0 + u * kPotrfThreads;
      if (idx < NB * NB) a[(idx / NB) * LD + idx % NB] = v[u];
    }
  }
  __syncthreads();
  POTRF_TICK(0);
  const int npan = (kb + kPanel - 1) / kPanel;
  for (int p = 0; p < npan; ++p) {
    const int c0 = p * kPanel;
    // ---- 1. warp 0: factor the 32 x 32 diagonal sub-block and invert it in
    // registers (lane i owns row i; columns move by shuffles, no block barrier)
    if (warp == 0) {
      // factor: lane i owns row i; column j of L goes straight to shared memory
      // and is read back by every lane as broadcasts (no shuffles but the pivot)
      double v[kPanel];
#pragma unroll
      for (int k = 0; k < kPanel; ++k) v[k] = a[(c0 + k) * LD + c0 + lane];  // k > lane: unused
      double myrs = 0.0;
      int firstbad = kPanel;
#pragma unroll
      for (int j = 0; j < kPanel; ++j) {
        double d = __shfl_sync(0xffffffffu, v[j], j);
        const bool bad = !(d > 0.0);
        firstbad = (bad && firstbad == kPanel) ? j : firstbad;
        d = bad ? 1.0 : d;  // continue (the launch sequence stays fixed); the factor is void
        const double rs = gbem_gpu::rsq64(d);
        const double lij = v[j] * rs;  // lane j: sqrt(d); lane i > j: L(i, j)
        myrs = lane == j ? rs : myrs;
        if (lane >= j) a[(c0 + j) * LD + c0 + lane] = lij;
        __syncwarp();
#pragma unroll
        for (int k = j + 1; k < kPanel; ++k) v[k] = fma(-lij, a[(c0 + j) * LD + c0 + k], v[k]);
      }
      if (lane == 0 && firstbad < kPanel && c0 + firstbad < kb) atomicMin(info, row0 + c0 + firstbad);
      xd[c0 + lane] = myrs;
      __syncwarp();
      // X = inv(L_pp): lane k owns column k (forward substitution, L broadcast
      // from shared memory): x_t = s_t / L_tt, then s_i -= L(i, t) x_t for i > t
      double x[kPanel];
#pragma unroll
      for (int i = 0; i < kPanel; ++i) x[i] = i == lane ? 1.0 : 0.0;
#pragma unroll
      for (int t = 0; t < kPanel; ++t) {
        x[t] *= xd[c0 + t];
#pragma unroll
        for (int i = t + 1; i < kPanel; ++i) x[i] = fma(-a[(c0 + t) * LD + c0 + i], x[t], x[i]);
      }
#pragma unroll
      for (int i = 0; i < kPanel; ++i)
        if (i > lane) a[(c0 + i) * LD + c0 + lane] = x[i];  // X(i, lane) in the strict upper half
    } else if ((warp & 3) != 0 && p > 0) {
      // the 12 warps off warp 0's sub-partition, in teams of two: the products
      // L_rq X_qp with q = p - 1 for every later block row r (<= 4 of them)
      const int slot = warp - 1 - (warp >> 2);  // 0..11 over warps 1,2,3,5,6,7,...
      const int team = slot >> 1, gt = (slot & 1) * 32 + lane;
      if (team < (npan - p) * p) potrf_inv_part1(a, xd, tmp, p + team / p, team % p, p - 1, gt);
      if (p == 3) POTRF_TICK_T(13, 64);
    }
    if (p == 3) POTRF_TICK(15);
    __syncthreads();
    POTRF_TICK(1 + 3 * p);
    const int r0 = c0 + kPanel, mrest = NB - r0;  // padded rows below the panel
    if (mrest <= 0) {
      // last panel: block row p of inv(L) on groups 0..p-1
      const int pb = tid >> 7;  // two 64-thread teams per block (row halves)
      POTRF_TICK(11);
      if (pb < p) potrf_inv_part2<2>(a, xd, tmp, p, pb, tid & 7, (tid >> 3) & 7, 2 * ((tid >> 6) & 1));
      POTRF_TICK(12);
      __syncthreads();
      break;
    }
    // Register tiles below are 4 x 4 with stride 8 inside 32 x 32 super-tiles of
    // 64 threads (tx, ty in 0..7: rows ty + 8u, columns tx + 8v), so that the
    // shared loads of a warp hit consecutive addresses or broadcast.
    const int grp = tid >> 6, tx = tid & 7, ty = (tid >> 3) & 7;
    // ---- 2. panel rows below: L_rp = A_rp * inv(L_pp)^T
    {
      const int G = mrest / kPanel;
      double acc[4][4] = {};
      const int rowb = r0 + kPanel * grp + ty;
      // groups 4..7 (two per block, row halves): block row p of inv(L) (rows < c0 of panel p's columns;
      // the panel rows below write rows >= r0 of the same columns)
      if (grp >= 4 && ((grp - 4) >> 1) < p) potrf_inv_part2<2>(a, xd, tmp, p, (grp - 4) >> 1, tx, ty, 2 * (grp & 1));
      if (grp < G) {
#pragma unroll 4
        for (int k = 0; k < kPanel; ++k) {  // X(j, k) = 0 for k > j: fixed trip count, no branches
          double ar[4], xv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) ar[u] = a[(c0 + k) * LD + rowb + 8 * u];
          const double dg = xd[c0 + k];
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int j = tx + 8 * v;
            const double up = a[(c0 + j) * LD + c0 + k];
            xv[v] = k < j ? up : 0.0;
            xv[v] = k == j ? dg : xv[v];  // X(j, k)
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] = fma(ar[u], xv[v], acc[u][v]);
        }
      }
      __syncthreads();
      if (grp < G) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) a[(c0 + tx + 8 * v) * LD + rowb + 8 * u] = acc[u][v];
      }
    }
    __syncthreads();
    POTRF_TICK(2 + 3 * p);
    // ---- 3. rank-32 update of the trailing lower part (32 x 32 super-tiles I >= J)
    {
      const int G = mrest / kPanel;
      if (grp < G * (G + 1) / 2) {
        int I = 0;
        while ((I + 1) * (I + 2) / 2 <= grp) ++I;
        const int J = grp - I * (I + 1) / 2;
        const int rowb = r0 + kPanel * I + ty, colb = r0 + kPanel * J + tx;
        double acc[4][4] = {};
#pragma unroll 4
        for (int k = 0; k < kPanel; ++k) {
          double lr[4], lc[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            lr[u] = a[(c0 + k) * LD + rowb + 8 * u];
            lc[u] = a[(c0 + k) * LD + colb + 8 * u];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] = fma(lr[u], lc[v], acc[u][v]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v)
            if (colb + 8 * v <= rowb + 8 * u) a[(colb + 8 * v) * LD + rowb + 8 * u] -= acc[u][v];
      }
    }
    __syncthreads();
    POTRF_TICK(3 + 3 * p);
  }
  POTRF_TICK(20);
  POTRF_TICK(21);
  // one pass: L (lower) back to A, X = inv(L) to Linv
  for (int idx = tid; idx < NB * NB; idx += kPotrfThreads) {
    const int c = idx / NB, r = idx % NB;  // constant divisor: shifts, not a division
    double v = 0.0;
    if (r < kb && c < kb) {
      if (r >= c) A[(long long)c * lda + r] = a[c * LD + r];
      if (r > c) v = a[r * LD + c];
      else if (r == c) v = xd[r];
    }
    Linv[c * NB + r] = v;
  }
  POTRF_TICK(22);
}

__global__ void k_save_diag(const double* A, long long lda, int n, double* d) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[i] = A[(long long)i * lda + i];
}

// y = A x with A given by its strict upper triangle (col-major, A[c*lda + r],
// r < c) and the saved diagonal.  One CTA per (64-row block, column chunk):
// it walks the 64 x 64 tiles of its rows, reading A(r, c) = A[c*lda + r] right
// of the diagonal and A(r, c) = A(c, r) = A[r*lda + c] left of it (both
// coalesced, staged into shared memory as [c][r]), and keeps y in registers;
// one atomic per (row, right-hand side, chunk).  Reads n^2 * 8 B (twice the
// stored triangle) but needs no per-tile atomics, which bound the symmetric
// one-pass form (~12M FP64 atomics at n = 11,340).
constexpr int kSymvChunks = 4;
template <int MAXR>
__global__ void __launch_bounds__(256) k_symv_upper(const double* __restrict__ A, long long lda,
                                                    const double* __restrict__ diag, int n, const double* X,
                                                    long long ldx, int nrhs, double* Y) {
  constexpr int T = 64, LD = T + 1;
  static_assert(MAXR % 2 == 0, "x rows read as double2");
  __shared__ double sa[T * LD];
  __shared__ __align__(16) double xs[T * MAXR];
  double* red = sa;  // [3][T][MAXR] quarter partials, after the tile loop
  static_assert(3 * T * MAXR <= T * LD, "partials fit in the tile buffer");
  const int nbt = (n + T - 1) / T;
  const int rb = blockIdx.x, r0 = rb * T;
  const int cb0 = (int)((long long)blockIdx.y * nbt / gridDim.y), cb1 = (int)((long long)(blockIdx.y + 1) * nbt / gridDim.y);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row = tid & (T - 1), quarter = tid >> 6;
  double acc[MAXR];
#pragma unroll
  for (int q = 0; q < MAXR; ++q) acc[q] = 0.0;
  // the tile of column block cb: column-wise right of (or on) the diagonal
  // (column c contiguous in r), row-wise left of it (A(r, c) = A[r*lda + c],
  // contiguous in c); the next tile's loads are in flight while this one is used
  auto load_tile = [&](int cb, double (&v)[T / 8][2]) {
    const int c0 = cb * T;
    if (cb >= rb) {
#pragma unroll
      for (int u = 0; u < T / 8; ++u) {
        const int c = c0 + warp + 8 * u;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = r0 + h * 32 + lane;
          v[u][h] = (c < n && r < c) ? __ldcs(A + (long long)c * lda + r) : 0.0;
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < T / 8; ++u) {
        const int r = r0 + warp + 8 * u;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = c0 + h * 32 + lane;
          v[u][h] = (r < n) ? __ldcs(A + (long long)r * lda + c) : 0.0;
        }
      }
    }
  };
  double v[T / 8][2], vn[T / 8][2];
  if (cb0 < cb1) load_tile(cb0, v);
  for (int cb = cb0; cb < cb1; ++cb) {
    const int c0 = cb * T;
    __syncthreads();  // the previous tile's reads of sa / xs are done
    if (cb >= rb) {
#pragma unroll
      for (int u = 0; u < T / 8; ++u)
#pragma unroll
        for (int h = 0; h < 2; ++h) sa[(warp + 8 * u) * LD + h * 32 + lane] = v[u][h];
    } else {
#pragma unroll
      for (int u = 0; u < T / 8; ++u)
#pragma unroll
        for (int h = 0; h < 2; ++h) sa[(h * 32 + lane) * LD + warp + 8 * u] = v[u][h];
    }
    for (int idx = tid; idx < T * MAXR; idx += 256) {
      const int c = idx % T, q = idx / T;
      xs[c * MAXR + q] = (q < nrhs && c0 + c < n) ? X[(long long)q * ldx + c0 + c] : 0.0;
    }
    if (cb + 1 < cb1) load_tile(cb + 1, vn);
    __syncthreads();
    if (cb == rb) {
      // diagonal tile: mirror the strict upper half into the lower, add the diagonal
      for (int idx = tid; idx < T * T; idx += 256) {
        const int c = idx / T, r = idx % T;
        if (r > c) sa[c * LD + r] = sa[r * LD + c];
        else if (r == c) sa[c * LD + r] = (r0 + r < n) ? diag[r0 + r] : 0.0;
      }
      __syncthreads();
    }
#pragma unroll 4
    for (int k = 0; k < T / 4; ++k) {
      const int c = quarter * (T / 4) + k;
      const double a = sa[c * LD + row];
      // x_c as 16-byte broadcasts (MAXR even)
      const double2* x2 = reinterpret_cast<const double2*>(xs + c * MAXR);
#pragma unroll
      for (int q = 0; q < MAXR / 2; ++q) {
        const double2 xv = x2[q];
        acc[2 * q] = fma(a, xv.x, acc[2 * q]);
        acc[2 * q + 1] = fma(a, xv.y, acc[2 * q + 1]);
      }
    }
#pragma unroll
    for (int u = 0; u < T / 8; ++u) {
      v[u][0] = vn[u][0];
      v[u][1] = vn[u][1];
    }
  }
  __syncthreads();  // last tile's reads of sa are done
  if (quarter > 0)
#pragma unroll
    for (int q = 0; q < MAXR; ++q) red[((quarter - 1) * T + row) * MAXR + q] = acc[q];
  __syncthreads();
  if (quarter == 0 && r0 + row < n) {
#pragma unroll
    for (int q = 0; q < MAXR; ++q) {
      const double y = acc[q] + red[(0 * T + row) * MAXR + q] + red[(1 * T + row) * MAXR + q] +
                       red[(2 * T + row) * MAXR + q];
      if (q < nrhs) atomicAdd(&Y[(long long)q * n + r0 + row], y);
    }
  }
}

// resid[q] = ||Y[:,q] - B[:,q]|| / ||B[:,q]|| (one CTA per rhs)
// Y = A X on the FP64 tensor cores for the residual, with A symmetric and only
// its strict upper triangle (col-major, A[c*lda + r], r < c) and the saved
// diagonal intact (the lower triangle holds L).  CTA: 64 rows of Y x NR
// right-hand sides, 4 warps of 16 x NR (2 x NR/8 DMMA m8n8k4 fragments); the
// reduction runs over all n columns in BK = 16 slabs, double-buffered by
// cp.async.  A slab right of the CTA's rows is read as stored (A(r, c) at
// c*lda + r, contiguous in r) into a [k][m] buffer, a slab left of them
// through the symmetry (A(r, c) = A[r*lda + c], contiguous in c) into an
// [m][k] buffer, and the few slabs crossing the diagonal element-wise; the
// fragment loads index whichever layout the slab used.  X (n x R, col-major)
// arrives as an [q][k] slab.  One pass over the matrix for up to NR
// right-hand sides (the scalar k_symv_upper streams it once per 8).
constexpr int kSyT = 64, kSyThreads = 128, kSyLU = kSyT + 8, kSyLL = BK + 4;
template <int NR>
struct SymmShape {
  static constexpr int LX = BK + 4;
  static constexpr int SLAB = BK * kSyLU + kSyT * kSyLL + NR * LX;  // upper layout, lower layout, X
  static constexpr size_t SMEM = 2 * SLAB * sizeof(double);
};
template <int NR>
__global__ void __launch_bounds__(kSyThreads, 4)
    k_symm_dmma(const double* __restrict__ A, long long lda, const double* __restrict__ diag, int n,
                const double* __restrict__ X, long long ldx, int R, double* __restrict__ Y) {
  using S = SymmShape<NR>;
  constexpr int FN = NR / 8;
  extern __shared__ __align__(16) double ssm[];
  const int r0 = blockIdx.x * kSyT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int nslab = (n + BK - 1) / BK;
  // slab kind: 0 upper (stored), 1 lower (transposed read), 2 crosses the diagonal
  auto kind = [&](int k0) { return k0 >= r0 + kSyT ? 0 : (k0 + BK <= r0 ? 1 : 2); };
  auto load = [&](int sl, int buf) {
    double* su = ssm + buf * S::SLAB;
    double* sL = su + BK * kSyLU;
    double* sx = sL + kSyT * kSyLL;
    const int k0 = sl * BK, kd = kind(k0);
    if (kd == 0) {
      for (int c = tid; c < BK * kSyT / 2; c += kSyThreads) {  // 16 columns x 64 rows, 16 B along r
        const int kk = c / (kSyT / 2), mm = (c % (kSyT / 2)) * 2;
        const int col = k0 + kk, row = r0 + mm;
        const bool ok = col < n && row < n;
        gbem_gemm::cp_async16(su + kk * kSyLU + mm, ok ? A + (long long)col * lda + row : A,
                              ok ? (row + 1 < n ? 16 : 8) : 0);
      }
    } else if (kd == 1) {
      for (int c = tid; c < kSyT * BK / 2; c += kSyThreads) {  // 64 rows x 16 columns, 16 B along c
        const int mm = c / (BK / 2), kk = (c % (BK / 2)) * 2;
        const int row = r0 + mm, col = k0 + kk;
        const bool ok = row < n && col < n;
        gbem_gemm::cp_async16(sL + mm * kSyLL + kk, ok ? A + (long long)row * lda + col : A,
                              ok ? (col + 1 < n ? 16 : 8) : 0);
      }
    } else {
      for (int e = tid; e < BK * kSyT; e += kSyThreads) {
        const int kk = e / kSyT, mm = e % kSyT;
        const int col = k0 + kk, row = r0 + mm;
        double v = 0.0;
        if (row < n && col < n)
          v = col > row ? A[(long long)col * lda + row] : (col < row ? A[(long long)row * lda + col] : diag[row]);
        su[kk * kSyLU + mm] = v;
      }
    }
    for (int c = tid; c < NR * BK / 2; c += kSyThreads) {  // X: NR columns x 16 rows, 16 B along k
      const int q = c / (BK / 2), kk = (c % (BK / 2)) * 2;
      const int col = k0 + kk;
      const bool ok = q < R && col < n;
      gbem_gemm::cp_async16(sx + q * S::LX + kk, ok ? X + (long long)q * ldx + col : X,
                            ok ? (col + 1 < n ? 16 : 8) : 0);
    }
    gbem_gemm::cp_async_commit();
  };
  double acc[2][FN][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  load(0, 0);
  for (int sl = 0; sl < nslab; ++sl) {
    if (sl + 1 < nslab) {
      load(sl + 1, (sl + 1) & 1);
      gbem_gemm::cp_async_wait<1>();
    } else {
      gbem_gemm::cp_async_wait<0>();
    }
    __syncthreads();
    const double* su = ssm + (sl & 1) * S::SLAB;
    const double* sL = su + BK * kSyLU;
    const double* sx = sL + kSyT * kSyLL;
    const bool lower = kind(sl * BK) == 1;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[2], bf[FN];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int m = warp * 16 + i * 8 + g;
        af[i] = lower ? sL[m * kSyLL + kk + t4] : su[(kk + t4) * kSyLU + m];
      }
#pragma unroll
      for (int j = 0; j < FN; ++j) bf[j] = sx[(j * 8 + g) * S::LX + kk + t4];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) gbem_gemm::dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int row = r0 + warp * 16 + i * 8 + g;
    if (row >= n) continue;
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int q = j * 8 + 2 * t4 + e;
        if (q < R) Y[(long long)q * n + row] = acc[i][j][e];
      }
  }
}

__global__ void k_resid_norm(const double* Y, const double* B, int n, double* resid) {
  int q = blockIdx.x;
  double rn = 0.0, bn = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double d = Y[(long long)q * n + i] - B[(long long)q * n + i];
    double b = B[(long long)q * n + i];
    rn += d * d;
    bn += b * b;
  }
  __shared__ double s1[1024], s2[1024];  // blockDim.x <= 1024, a power of two
  s1[threadIdx.x] = rn;
  s2[threadIdx.x] = bn;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      s1[threadIdx.x] += s1[threadIdx.x + o];
      s2[threadIdx.x] += s2[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double b = sqrt(s2[0]);
    resid[q] = sqrt(s1[0]) / (b > 0.0 ? b : 1.0);
  }
}


// Forward (L Y = B) and backward (L^T X = Y) block substitution for up to
// kSolveR right-hand sides in one cooperative launch (one CTA per SM).
// Step k: the 128 x 128 diagonal-block inverse inv(L_kk) sits in shared memory
// (cp.async prefetch of the next block overlaps the current step); every CTA
// forms y = inv(L_kk) w_k (or inv(L_kk)^T) redundantly, CTA 0 publishes it, and
// each CTA updates the rows it owns (a fixed range of 32-row strips) below
// (forward) or above (backward) the block; one grid barrier per step.
// The factor entries a step needs do not depend on the solution, so each CTA
// issues the loads of its first kSolvePF strips of the NEXT step's panel before
// the grid barrier: the DRAM latency of the panel overlaps the barrier and the
// diagonal solve, and a step costs ~ barrier + diagonal solve.
// Buffers: W = B copy that receives the forward updates and finally the
// solution X; Out = forward results Y that receive the backward updates.
constexpr int kSolveThreads = 256;
constexpr int kSolveWarps = kSolveThreads / 32;
constexpr int kSolveR = 16;
constexpr int kSolvePF = 3;                      // register-prefetched strips per CTA and step
constexpr int kSolveCols = NB / kSolveWarps;     // forward: block columns per warp (16)
static_assert(kSolveCols == 16 && NB / 32 == 4, "strip tiling assumes NB = 128, 8 warps");
// The diagonal-block inverse sits in shared memory with column stride NB + 2
// (16-byte aligned columns; column reads (forward) and row reads (backward,
// the transposed product) are both at most 2-way bank conflicted).
constexpr int kLsLd = NB + 2;
constexpr size_t kSolveSmem =
    (size_t)(NB * kLsLd + 3 * kSolveR * NB + kSolveWarps * kSolveR * 32 + kSolvePF * kSolveR * 32) * sizeof(double);

__device__ __forceinline__ void solve_prefetch_block(double* Ls, const double* Li, int tid) {
  for (int c = tid; c < NB * NB / 2; c += kSolveThreads) {
    const int col = (2 * c) / NB, row = (2 * c) % NB;
    unsigned s = (unsigned)__cvta_generic_to_shared(Ls + col * kLsLd + row);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(Li + 2 * c));
  }
  asm volatile("cp.async.commit_group;\n" ::);
}

// ys[q][i] = sum_kk M(i,kk) ws[q][kk] with M = inv(L) (transpose = 0, kk <= i) or
// inv(L)^T (transpose = 1, kk >= i); two threads per row i, partial sums folded in smem.
template <int RT>
__device__ __forceinline__ void solve_diag(const double* Ls, const double* ws, double* ys, double* part, int kb,
                                          int R, int transpose, int tid) {
  static_assert(2 * NB == kSolveThreads, "two threads per diagonal-block row");
  const int i = tid % NB, half = tid / NB;
  double acc[RT];
#pragma unroll
  for (int q = 0; q < RT; ++q) acc[q] = 0.0;
  if (i < kb) {
    const int lo = transpose ? i : 0, hi = transpose ? kb : i + 1;
    const int mid = (lo + hi) >> 1;
    const int b0 = half ? mid : lo, b1 = half ? hi : mid;
#pragma unroll 4
    for (int kk = b0; kk < b1; ++kk) {
      const double m = transpose ? Ls[i * kLsLd + kk] : Ls[kk * kLsLd + i];
#pragma unroll
      for (int q = 0; q < RT; ++q)
        if (q < R) acc[q] = fma(m, ws[q * NB + kk], acc[q]);
    }
  }
  if (half)
#pragma unroll
    for (int q = 0; q < RT; ++q)
      if (q < R) part[q * NB + i] = acc[q];
  __syncthreads();
  // Every ys slot strip_update reads is written: rows >= kb of a ragged last
  // block and columns q >= R are zero (fma(0, leftover NaN) would poison T).
  if (!half)
#pragma unroll
    for (int q = 0; q < RT; ++q) ys[q * NB + i] = (i < kb && q < R) ? acc[q] + part[q * NB + i] : 0.0;
  __syncthreads();
}

// Forward panel loads of strip s for block (k0, kb): lane = row 32 s + lane,
// warp w = block columns [16 w, 16 w + 16) (coalesced 256 B per instruction).
__device__ __forceinline__ void fwd_load(const double* __restrict__ A, long long lda, int n, int k0, int kb, int s,
                                         int warp, int lane, double (&l)[kSolveCols]) {
  const long long r = 32LL * s + lane;
#pragma unroll
  for (int u = 0; u < kSolveCols; ++u) {
    const int c = warp * kSolveCols + u;
    l[u] = (r < n && c < kb) ? __ldcs(A + (long long)(k0 + c) * lda + r) : 0.0;
  }
}
// Backward panel loads of strip s: lane = row r = 32 s + lane of L^T, i.e.
// column r of L, whose block entries L(k0 + c, r) = A[r * lda + k0 + c] are
// contiguous in c: warp w reads c in [16 w, 16 w + 16) as eight 16-byte loads
// (one 128-byte line per lane; k0 + 16 w is a multiple of 16, lda of 8).
__device__ __forceinline__ void bwd_load(const double* __restrict__ A, long long lda, int k0, int kb, int s,
                                         int warp, int lane, double (&l)[kSolveCols]) {
  const long long r = 32LL * s + lane;
  const double2* src = reinterpret_cast<const double2*>(A + r * lda + k0 + warp * kSolveCols);
#pragma unroll
  for (int u = 0; u < kSolveCols / 2; ++u) {
    const int c = warp * kSolveCols + 2 * u;
    const double2 v = c < kb ? __ldcs(src + u) : make_double2(0.0, 0.0);
    l[2 * u] = v.x;
    l[2 * u + 1] = c + 1 < kb ? v.y : 0.0;
  }
}

// T[q][r] -= sum_c P(r, c) y[q][c] for the nk strips c0.. of this CTA: lane = row,
// warp = 16 block columns (pf), cross-warp sums through `red`, then one
// read-modify-write pass over the chunk with every load issued before any store.
template <int RT>
__device__ __forceinline__ void strip_update(const double (&pf)[kSolvePF][kSolveCols], const double* ys, double* red,
                                             double* vb, double* T, int n, int R, int c0, int nk, int tid, int warp,
                                             int lane) {
#pragma unroll
  for (int k = 0; k < kSolvePF; ++k) {
    if (k >= nk) break;
    double acc[RT];
#pragma unroll
    for (int q = 0; q < RT; ++q) acc[q] = 0.0;
#pragma unroll
    for (int u = 0; u < kSolveCols; ++u) {
      const int c = warp * kSolveCols + u;
#pragma unroll
      for (int q = 0; q < RT; ++q) acc[q] = fma(pf[k][u], ys[q * NB + c], acc[q]);
    }
#pragma unroll
    for (int q = 0; q < RT; ++q) red[(warp * RT + q) * 32 + lane] = acc[q];
    __syncthreads();
    for (int idx = tid; idx < 32 * R; idx += kSolveThreads) {
      double v = 0.0;
#pragma unroll
      for (int w = 0; w < kSolveWarps; ++w) v += red[w * RT * 32 + idx];
      vb[k * RT * 32 + idx] = v;
    }
    __syncthreads();
  }
  constexpr int kIt = (kSolvePF * RT * 32 + kSolveThreads - 1) / kSolveThreads;
  double old[kIt];
  long long addr[kIt];
#pragma unroll
  for (int t = 0; t < kIt; ++t) {
    const int idx = tid + t * kSolveThreads, k = idx / (32 * RT), q = (idx / 32) % RT, ln = idx % 32;
    const long long r = 32LL * (c0 + k) + ln;
    addr[t] = (k < nk && q < R && r < n) ? (long long)q * n + r : -1;
    old[t] = addr[t] >= 0 ? T[addr[t]] : 0.0;
  }
#pragma unroll
  for (int t = 0; t < kIt; ++t) {
    const int idx = tid + t * kSolveThreads, k = idx / (32 * RT), q = (idx / 32) % RT, ln = idx % 32;
    if (addr[t] >= 0) T[addr[t]] = old[t] - vb[(k * RT + q) * 32 + ln];
  }
}

#ifdef GBEM_SOLVE_TIMING
__device__ long long g_solve_clk[2][8];
#define SOLVE_TICK(slot)                                                          \
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x / 2)) {    \
    long long t_ = clock64();                                                     \
    g_solve_clk[blockIdx.x == 0 ? 0 : 1][slot] += t_ - t_prev;                    \
    t_prev = t_;                                                                  \
  }
#else
#define SOLVE_TICK(slot)
#endif
template <int RT>
__global__ void __launch_bounds__(kSolveThreads, 1)
    k_solve_coop(const double* __restrict__ A, long long lda, const double* __restrict__ Linv, int n, int R,
                 const double* __restrict__ B, double* W, double* Out, int dbg) {
  // dbg (phase-breakdown timing only, GBEM_SOLVE_DBG): 1 skip diagonal solves,
  // 2 skip panel updates, 4 skip grid barriers (results wrong for 1/2/4)
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sm[];
  double* Ls = sm;                    // [NB][NB] current diagonal-block inverse
  double* ws = Ls + NB * kLsLd;       // [RT][NB] right-hand side block
  double* ys = ws + RT * NB;     // [RT][NB] solved block
  double* part = ys + RT * NB;   // [RT][NB] partial sums
  double* red = part + RT * NB;  // [warps][RT][32] forward cross-warp sums
  double* vb = red + kSolveWarps * RT * 32;  // [kSolvePF][RT][32] reduced strip updates
  const int nblk = (n + NB - 1) / NB;
  const int nstrips = (n + 31) / 32;
  const int s_lo = (int)((long long)blockIdx.x * nstrips / gridDim.x);
  const int s_hi = (int)((long long)(blockIdx.x + 1) * nstrips / gridDim.x);
  const long long nR = (long long)n * R;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double pf[kSolvePF][kSolveCols];

  // first owned strip strictly below block b (k0 + kb is a multiple of 32 or n)
  auto fwd_first = [&](int b) {
    const int k0 = b * NB, kb = min(NB, n - k0);
    return max(s_lo, (k0 + kb + 31) / 32);
  };
  auto fwd_prefetch = [&](int b) {
    const int k0 = b * NB, kb = min(NB, n - k0), s0 = fwd_first(b);
#pragma unroll
    for (int k = 0; k < kSolvePF; ++k)
      if (s0 + k < s_hi) fwd_load(A, lda, n, k0, kb, s0 + k, warp, lane, pf[k]);
  };
  auto bwd_prefetch = [&](int b) {
    const int k0 = b * NB, kb = min(NB, n - k0), s1 = min(s_hi, k0 / 32);
#pragma unroll
    for (int k = 0; k < kSolvePF; ++k)
      if (s_lo + k < s1) bwd_load(A, lda, k0, kb, s_lo + k, warp, lane, pf[k]);
  };

#ifdef GBEM_SOLVE_TIMING
  long long t_prev = clock64();
#endif
  solve_prefetch_block(Ls, Linv, tid);
  fwd_prefetch(0);
  for (long long i = grid.thread_rank(); i < nR; i += grid.size()) W[i] = B[i];
  grid.sync();
  // ---- forward: W holds b - sum_{j<k} L_kj y_j, Out receives y
  for (int b = 0; b < nblk; ++b) {
    const int k0 = b * NB, kb = min(NB, n - k0);
    for (int idx = tid; idx < kb * R; idx += blockDim.x) {
      const int i = idx % kb, q = idx / kb;
      ws[q * NB + i] = W[(long long)q * n + k0 + i];
    }
    SOLVE_TICK(0);
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
    SOLVE_TICK(1);
    const int s0 = fwd_first(b);
    const bool active = s0 < s_hi;
    if ((active || blockIdx.x == 0) && !(dbg & 1)) solve_diag<RT>(Ls, ws, ys, part, kb, R, 0, tid);
    SOLVE_TICK(2);
    solve_prefetch_block(Ls, Linv + (size_t)min(b + 1, nblk - 1) * NB * NB, tid);  // backward starts at the last
    if (blockIdx.x == 0)
      for (int idx = tid; idx < kb * R; idx += blockDim.x) {
        const int i = idx % kb, q = idx / kb;
        Out[(long long)q * n + k0 + i] = ys[q * NB + i];
      }
    for (int c0 = s0; c0 < ((dbg & 2) ? s0 : s_hi); c0 += kSolvePF) {
      if (c0 != s0) {
#pragma unroll
        for (int k = 0; k < kSolvePF; ++k)
          if (c0 + k < s_hi) fwd_load(A, lda, n, k0, kb, c0 + k, warp, lane, pf[k]);
      }
      strip_update<RT>(pf, ys, red, vb, W, n, R, c0, min(kSolvePF, s_hi - c0), tid, warp, lane);
    }
    SOLVE_TICK(3);
    if (b + 1 < nblk) fwd_prefetch(b + 1);
    else bwd_prefetch(nblk - 1);
    SOLVE_TICK(4);
    if (!(dbg & 4)) grid.sync();
    SOLVE_TICK(5);
  }
  // ---- backward: Out holds y - sum_{j>k} L_jk^T x_j, W receives x
  for (int b = nblk - 1; b >= 0; --b) {
    const int k0 = b * NB, kb = min(NB, n - k0);
    for (int idx = tid; idx < kb * R; idx += blockDim.x) {
      const int i = idx % kb, q = idx / kb;
      ws[q * NB + i] = Out[(long long)q * n + k0 + i];
    }
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
    const int s1 = min(s_hi, k0 / 32);
    const bool active = s_lo < s1;
    if ((active || blockIdx.x == 0) && !(dbg & 1)) solve_diag<RT>(Ls, ws, ys, part, kb, R, 1, tid);
    if (b > 0) solve_prefetch_block(Ls, Linv + (size_t)(b - 1) * NB * NB, tid);
    if (blockIdx.x == 0)
      for (int idx = tid; idx < kb * R; idx += blockDim.x) {
        const int i = idx % kb, q = idx / kb;
        W[(long long)q * n + k0 + i] = ys[q * NB + i];
      }
    // rows r < k0: Out[r] -= sum_{c in block} L(k0+c, r) x_c
    for (int c0 = s_lo; c0 < ((dbg & 2) ? s_lo : s1); c0 += kSolvePF) {
      if (c0 != s_lo) {
#pragma unroll
        for (int k = 0; k < kSolvePF; ++k)
          if (c0 + k < s1) bwd_load(A, lda, k0, kb, c0 + k, warp, lane, pf[k]);
      }
      strip_update<RT>(pf, ys, red, vb, Out, n, R, c0, min(kSolvePF, s1 - c0), tid, warp, lane);
    }
    if (b > 0) bwd_prefetch(b - 1);
    if (!(dbg & 4)) grid.sync();
  }
}

// Backward substitution L^T X = Y as a dataflow over the 128-row blocks, for
// the bordered factorisation (Y from the border rows).  CTA b owns block b:
//   X_b = inv(L_bb)^T (Y_b - sum_{c > b} L_cb^T X_c)
// in the left-looking (dot-product) form, walking c = nblk-1 .. b+1.  The
// 128 x 128 block L_cb is staged in shared memory by coalesced cp.async
// (its load is issued before the CTA waits for the flag of X_c, so the L
// stream, n^2/2 * 8 B over all CTAs, overlaps the dependency chain); the
// diagonal-block inverse sits in registers from the start.  The chain per
// block is one X_c hand-off (release / acquire flag), a 128 x 128 x R product
// from shared memory and the diagonal solve -- no grid barrier.  Thread
// (i, h): column i of the block, rows [64 h, 64 h + 64).  One CTA per block,
// all co-resident (cooperative launch), nblk <= #SMs.
constexpr int kFlowThreads = 256, kFlowLD = NB + 1;
constexpr size_t kFlowSmem = (size_t)(NB * kFlowLD + 3 * NB * 16) * sizeof(double);
template <int RT>
__global__ void __launch_bounds__(kFlowThreads, 1)
    k_bwd_flow(const double* __restrict__ A, long long lda, const double* __restrict__ Linv, int n, int R,
               const double* __restrict__ Y, double* X, int* flags, int epoch) {
  extern __shared__ __align__(16) double fsm[];
  double* Lb = fsm;                       // [row r][col i] of L_cb, ld kFlowLD
  double* xs = Lb + NB * kFlowLD;         // [r][RT]
  double* red = xs + NB * RT;             // [i][RT] half-1 partials
  double* ys = red + NB * RT;             // [k][RT]
  const int b = blockIdx.x, nblk = gridDim.x;
  const int k0 = b * NB, kb = min(NB, n - k0);
  const int tid = threadIdx.x, i = tid & (NB - 1), h = tid >> 7;
  // inv(L_bb)(k, i) for k in [64 h, 64 h + 64): column i of the inverse (contiguous)
  double dinv[64];
  {
    const double* li = Linv + (size_t)b * NB * NB + (size_t)i * NB + 64 * h;
#pragma unroll
    for (int k = 0; k < 64; ++k) dinv[k] = li[k];
  }
  double acc[RT], yb[RT];  // yb: Y_b(i), loaded off the dependency chain
#pragma unroll
  for (int q = 0; q < RT; ++q) {
    acc[q] = 0.0;
    yb[q] = (h == 0 && i < kb && q < R) ? Y[(long long)q * n + k0 + i] : 0.0;
  }
  auto issue_block = [&](int c) {  // L(c0 + r, k0 + i) -> Lb[r][i], zero outside the matrix
    const int c0 = c * NB, kc = min(NB, n - c0);
    for (int idx = tid; idx < NB * NB; idx += kFlowThreads) {
      const int r = idx & (NB - 1), col = idx >> 7;
      const bool ok = r < kc && col < kb;
      gbem_gemm::cp_async8(Lb + r * kFlowLD + col, ok ? A + (long long)(k0 + col) * lda + c0 + r : A, ok ? 8 : 0);
    }
    gbem_gemm::cp_async_commit();
  };
  if (b + 1 < nblk) issue_block(nblk - 1);
  for (int c = nblk - 1; c > b; --c) {
    const int c0 = c * NB, kc = min(NB, n - c0);
    if (tid == 0) {
      // relaxed polls (an acquire load per poll also invalidates L1 each time),
      // then one acquire fence; X_c is read through L2 below
      int f;
      do {
        asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(f) : "l"(flags + c) : "memory");
      } while (f != epoch);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
    for (int idx = tid; idx < NB * RT; idx += kFlowThreads) {
      const int r = idx / RT, q = idx % RT;
      xs[idx] = (q < R && r < kc) ? __ldcg(X + (long long)q * n + c0 + r) : 0.0;
    }
    gbem_gemm::cp_async_wait<0>();
    __syncthreads();
#pragma unroll 8
    for (int r = 0; r < 64; ++r) {
      const double l = Lb[(64 * h + r) * kFlowLD + i];
#pragma unroll
      for (int q = 0; q < RT; ++q) acc[q] = fma(l, xs[(64 * h + r) * RT + q], acc[q]);
    }
    __syncthreads();  // Lb and xs are reused
    if (c - 1 > b) issue_block(c - 1);
  }
  // y = Y_b - (both row halves)
  if (h == 1)
#pragma unroll
    for (int q = 0; q < RT; ++q) red[i * RT + q] = acc[q];
  __syncthreads();
  if (h == 0)
#pragma unroll
    for (int q = 0; q < RT; ++q)
      ys[i * RT + q] = (i < kb && q < R) ? yb[q] - (acc[q] + red[i * RT + q]) : 0.0;
  __syncthreads();
  // X_b(i) = sum_k inv(L_bb)(k, i) y_k (the inverse is zero above its diagonal)
  double o[RT];
#pragma unroll
  for (int q = 0; q < RT; ++q) o[q] = 0.0;
#pragma unroll
  for (int k = 0; k < 64; ++k)
#pragma unroll
    for (int q = 0; q < RT; ++q) o[q] = fma(dinv[k], ys[(64 * h + k) * RT + q], o[q]);
  if (h == 1)
#pragma unroll
    for (int q = 0; q < RT; ++q) red[i * RT + q] = o[q];
  __syncthreads();
  if (h == 0 && i < kb)
#pragma unroll
    for (int q = 0; q < RT; ++q)
      if (q < R) X[(long long)q * n + k0 + i] = o[q] + red[i * RT + q];
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(flags + b), "r"(epoch) : "memory");
  }
}

// Column-major (R x n, ld n: one right-hand side per column of the caller's
// layout) <-> row-major (n x R: the R values of a panel contiguous).
__global__ void k_rhs_transpose(const double* __restrict__ in, int n, int R, double* __restrict__ out, int to_rows,
                                int ldr = 0) {
  if (ldr == 0) ldr = R;  // row stride of the row-major side
  __shared__ double t[32][33];
  const int i0 = blockIdx.x * 32, q0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int k = ty; k < 32; k += 8) {
    const int i = i0 + tx, q = q0 + k;  // read coalesced along i (column-major source)
    if (to_rows) t[k][tx] = (i < n && q < R) ? in[(long long)q * n + i] : 0.0;
    else {
      const int ii = i0 + k, qq = q0 + tx;  // row-major source: coalesced along q
      t[k][tx] = (ii < n && qq < R) ? in[(long long)ii * ldr + qq] : 0.0;
    }
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    if (to_rows) {
      const int i = i0 + k, q = q0 + tx;
      if (i < n && q < R) out[(long long)i * ldr + q] = t[tx][k];
    } else {
      const int q = q0 + k, i = i0 + tx;
      if (i < n && q < R) out[(long long)q * n + i] = t[tx][k];
    }
  }
}

}  // namespace

// y of the bordered factorisation: border row n + q of column c holds Y(c, q).
// rowmajor: Y[c * R + q] (blocked solve), else Y[q * n + c] (cooperative solve).
__global__ void k_border_to_y(const double* __restrict__ A, long long lda, int n, int R, double* __restrict__ Y,
                              int rowmajor) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)n * R) return;
  const long long c = i / R;
  const int q = (int)(i % R);
  const double v = A[c * lda + n + q];
  if (rowmajor)
    Y[i] = v;
  else
    Y[(long long)q * n + c] = v;
}

// Blocked forward/backward substitution on the FP64 tensor cores for wide
// right-hand-side blocks (R >= 17): the right-hand sides in row-major n x R
// form W, then per 128-block b
//   forward   Y_b^T = W_b^T inv(L_bb)^T             (k_gemm_g<kStore, NT>)
//             W_below^T -= Y_b^T L_below,b^T         (k_gemm_g<kSub, NT>)
//   backward  X_b^T = Y_b^T inv(L_bb)                (k_gemm_g<kStore, NN>)
//             Y_above^T -= X_b^T L_b,above           (k_gemm_g<kSub, NN>)
// 2 n^2 R flops per solve on DMMA instead of the latency-bound cooperative
// kernel (whose per-step cost grows with R).
static int solve_blocked(gbem_ctx* ctx, const double* d_B, int R, double* d_X, bool y_from_border) {
  const int n = (int)ctx->n;
  const long long lda = ctx->lda;
  cudaStream_t s = ctx->stream;
  const size_t nr = (size_t)n * R;
  if (ctx->sw_cap < 3 * nr) {
    cudaFree(ctx->d_sw);
    ctx->d_sw = nullptr;
    ctx->sw_cap = 0;
    GBEM_CUDA(ctx, cudaMalloc(&ctx->d_sw, 3 * nr * sizeof(double)));
    ctx->sw_cap = 3 * nr;
  }
  double* W = ctx->d_sw;
  double* Y = W + nr;
  double* X = Y + nr;
  if (!(ctx->attr_set & gbem_ctx::kAttrGemmSolve)) {
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_gemm_g<kStore, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGSmem));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_gemm_g<kSub, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGSmem));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_gemm_g<kStore, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGSmem));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_gemm_g<kSub, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGSmem));
    ctx->attr_set |= gbem_ctx::kAttrGemmSolve;
  }
  const dim3 tb(32, 8), tg((n + 31) / 32, (R + 31) / 32);
  if (y_from_border) {
    const long long cnt = (long long)n * R;
    k_border_to_y<<<(unsigned)((cnt + 255) / 256), 256, 0, s>>>(ctx->d_A, lda, n, R, Y, 1);
  } else {
    k_rhs_transpose<<<tg, tb, 0, s>>>(d_B, n, R, W, 1);
  }
  GBEM_LAUNCH_CHECK(ctx);
  const double* L = ctx->d_A;
  const double* Linv = ctx->d_linv;
  const int vec = (R % 2 == 0 && lda % 2 == 0) ? 1 : 0;
  const int nblk = (n + NB - 1) / NB;
  const unsigned gm = (unsigned)((R + kGT - 1) / kGT);
  for (int b = 0; b < (y_from_border ? 0 : nblk); ++b) {
    const int k0 = b * NB, kb = std::min(NB, n - k0), m = n - k0 - kb;
    const double* Lbb = Linv + (size_t)b * NB * NB;
    k_gemm_g<kStore, 0><<<dim3(gm, (kb + kGT - 1) / kGT), kGThreads, kGSmem, s>>>(
        Y + (size_t)k0 * R, R, W + (size_t)k0 * R, R, Lbb, NB, R, kb, kb, vec);
    GBEM_LAUNCH_CHECK(ctx);
    if (m > 0) {
      k_gemm_g<kSub, 0><<<dim3(gm, (m + kGT - 1) / kGT), kGThreads, kGSmem, s>>>(
          W + (size_t)(k0 + kb) * R, R, Y + (size_t)k0 * R, R, L + (long long)k0 * lda + k0 + kb, lda, R, m, kb, vec);
      GBEM_LAUNCH_CHECK(ctx);
    }
  }
  for (int b = nblk - 1; b >= 0; --b) {
    const int k0 = b * NB, kb = std::min(NB, n - k0);
    const double* Lbb = Linv + (size_t)b * NB * NB;
    k_gemm_g<kStore, 1><<<dim3(gm, (kb + kGT - 1) / kGT), kGThreads, kGSmem, s>>>(
        X + (size_t)k0 * R, R, Y + (size_t)k0 * R, R, Lbb, NB, R, kb, kb, vec);
    GBEM_LAUNCH_CHECK(ctx);
    if (k0 > 0) {
      k_gemm_g<kSub, 1><<<dim3(gm, (k0 + kGT - 1) / kGT), kGThreads, kGSmem, s>>>(
          Y, R, X + (size_t)k0 * R, R, L + k0, lda, R, k0, kb, vec);
      GBEM_LAUNCH_CHECK(ctx);
    }
  }
  k_rhs_transpose<<<tg, tb, 0, s>>>(X, n, R, d_X, 0);
  GBEM_LAUNCH_CHECK(ctx);
  return GBEM_OK;
}

// ---------------------------------------------------------------------------
// Look-ahead backward substitution L^T X = Y for the bordered extraction with
// 17..64 right-hand sides.  The plain blocked sweep above runs two dependent
// launches per 128-row block (31 us per block on config 3: latency, not HBM).
// Here the dependency chain and the bulk of the work are separated:
//   chain (high-priority stream), one 8-CTA cluster launch per block b:
//     X_b = inv(L_bb)^T (Y1_b + Y2_b);   Y1_{b-1} -= L_{b,b-1}^T X_b
//   bulk (the caller's stream), one DMMA GEMM per block b:
//     Y2_{0..b-2} -= L_{b,0..b-2}^T X_b
// Y1 is only touched by the chain and Y2 only by the bulk stream, so the two never
// write the same rows; step b waits for bulk(b + 2), which had a whole step to
// finish.  In the step kernel cluster rank r owns 16 of the block's 128 columns:
// its slabs of inv(L_bb) and L_{b,b-1} are staged by cp.async before anything that
// depends on the previous step, the 16 x R slice of X_b is written to every CTA of
// the cluster through distributed shared memory, and after one cluster barrier the
// same CTA forms its 16 rows of the Y1_{b-1} update.  Work arrays are row-major
// n x Rs (Rs = R rounded up to even: 16-byte cp.async in the bulk GEMM).
constexpr int kStepCluster = 8, kStepThreads = 512, kStepCols = NB / kStepCluster, kStepKG = 8;
// shared-memory strides (doubles) that spread the DMMA fragment loads over all banks: slab rows
// (k contiguous) = 4 mod 16, right-hand-side rows (m contiguous) = 8 mod 16
constexpr int kSlabLd = NB + 4;
constexpr int kStepRMax = 64;
__host__ __device__ constexpr int rhs_stride(int NF) { return NF % 2 ? 8 * NF : 8 * NF + 8; }
static int rhs_frags(int Rs) { return Rs <= 8 ? 1 : Rs <= 16 ? 2 : Rs <= 24 ? 3 : Rs <= 32 ? 4 : Rs <= 48 ? 6 : 8; }
static size_t step_smem(int NF) { return (size_t)(2 * kStepCols * kSlabLd + 2 * NB * rhs_stride(NF)) * sizeof(double); }

// y of the bordered factorisation as rows of stride Rs (columns >= R zero)
__global__ void k_border_to_rows(const double* __restrict__ A, long long lda, int n, int R, int Rs,
                                 double* __restrict__ Y) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)n * Rs) return;
  const long long c = i / Rs;
  const int q = (int)(i % Rs);
  Y[i] = q < R ? A[c * lda + n + q] : 0.0;
}

// acc (8 slab rows x 8 NF right-hand sides) += slab rows (k in [k0, k0 + 4 ksteps)) * V rows:
// a = this lane's slab element (row g, k0 + t4), v = V + (k0 + t4) * Vs + g
template <int NF>
__device__ __forceinline__ void dmma_rows(const double* __restrict__ a, const double* __restrict__ v, int Vs, int ksteps,
                                          double (&acc)[NF][2]) {
#pragma unroll 4
  for (int ks = 0; ks < ksteps; ++ks) {
    const double av = a[4 * ks];
#pragma unroll
    for (int f = 0; f < NF; ++f) dmma(acc[f][0], acc[f][1], av, v[4 * ks * Vs + 8 * f]);
  }
}

// rows [r0, r0 + rows) of a row-major (rows x Rs) global block into shared rows of stride Vs
// (16-byte cp.async; Rs even), rows >= live zero-filled
__device__ __forceinline__ void stage_rows(double* dst, int Vs, const double* src, int Rs, int live, int tid, int nthreads) {
  const int cpr = Rs / 2;  // 16-byte chunks per row
  for (int c = tid; c < NB * cpr; c += nthreads) {
    const int r = c / cpr, q = 2 * (c % cpr);
    cp_async16(&dst[r * Vs + q], r < live ? src + (size_t)r * Rs + q : src, r < live ? 16 : 0);
  }
}

template <int NF>  // 8-wide right-hand-side fragments (Rs <= 8 NF)
__global__ void __cluster_dims__(kStepCluster, 1, 1) __launch_bounds__(kStepThreads)
    k_bwd_step(const double* __restrict__ Linv_b, const double* __restrict__ L, long long lda, double* Y1,
               const double* Y2, double* X, int Rs, int k0, int kb) {
  constexpr int Vs = rhs_stride(NF);
  extern __shared__ __align__(16) double smem[];
  double* Ai = smem;                      // [16][kSlabLd]: Ai[j][k] = inv(L_bb)(k, j0 + j)
  double* Lb = Ai + kStepCols * kSlabLd;  // [16][kSlabLd]: Lb[j][k] = L(k0 + k, k0 - NB + j0 + j)
  double* T = Lb + kStepCols * kSlabLd;   // [NB][Vs]: Y1_b + Y2_b; then the partial sums red[kg][16][8 NF]
  double* Xs = T + NB * Vs;               // [NB][Vs]: X_b, gathered from the cluster
  double* red = T;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int nf = warp & 1, kg = warp >> 1;  // this warp: slab rows [8 nf, 8 nf + 8), k in [16 kg, 16 kg + 16)
  const int j0 = rank * kStepCols;
  // everything this step reads is requested at once: the two slabs (they do not depend on
  // the previous step) and Y1_b by cp.async, Y2_b into registers
  for (int c = tid; c < kStepCols * (NB / 2); c += kStepThreads) {
    const int jj = c / (NB / 2), k = 2 * (c % (NB / 2));
    const bool ok1 = k < kb && j0 + jj < kb;
    cp_async16(&Ai[jj * kSlabLd + k], ok1 ? Linv_b + (size_t)(j0 + jj) * NB + k : Linv_b,
               ok1 ? (k + 1 < kb ? 16 : 8) : 0);
    const bool ok2 = k0 > 0 && k < kb;
    cp_async16(&Lb[jj * kSlabLd + k], ok2 ? L + (long long)(k0 - NB + j0 + jj) * lda + k0 + k : L,
               ok2 ? (k + 1 < kb ? 16 : 8) : 0);
  }
  stage_rows(T, Vs, Y1 + (size_t)k0 * Rs, Rs, kb, tid, kStepThreads);
  cp_async_commit();
  double y2[2 * NF];
#pragma unroll
  for (int u = 0; u < 2 * NF; ++u) {
    const int c = tid + u * kStepThreads;
    y2[u] = c < kb * Rs ? Y2[(size_t)k0 * Rs + c] : 0.0;
  }
  for (int c = tid; c < NB * (Vs - Rs); c += kStepThreads) {  // zero the padding columns of T and Xs
    const int r = c / (Vs - Rs), q = Rs + c % (Vs - Rs);
    T[r * Vs + q] = 0.0;
    Xs[r * Vs + q] = 0.0;
  }
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 2 * NF; ++u) {
    const int c = tid + u * kStepThreads;
    if (c < NB * Rs) T[(c / Rs) * Vs + c % Rs] += y2[u];
  }
  __syncthreads();
  // x(j0 + j, m) = sum_k inv(L_bb)(k, j0 + j) T(k, m)  (zero for rows >= kb: zero-filled slab)
  double acc[NF][2];
#pragma unroll
  for (int f = 0; f < NF; ++f) acc[f][0] = acc[f][1] = 0.0;
  dmma_rows<NF>(Ai + (8 * nf + g) * kSlabLd + 16 * kg + t4, T + (16 * kg + t4) * Vs + g, Vs, 4, acc);
  __syncthreads();  // T is dead: its space takes the partial sums
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    red[(kg * kStepCols + 8 * nf + g) * (8 * NF) + 8 * f + 2 * t4] = acc[f][0];
    red[(kg * kStepCols + 8 * nf + g) * (8 * NF) + 8 * f + 2 * t4 + 1] = acc[f][1];
  }
  __syncthreads();
  for (int o = tid; o < kStepCols * Rs; o += kStepThreads) {
    const int jj = o / Rs, m = o % Rs;
    double x = 0.0;
#pragma unroll
    for (int q = 0; q < kStepKG; ++q) x += red[(q * kStepCols + jj) * (8 * NF) + m];
    if (j0 + jj < kb) X[(size_t)(k0 + j0) * Rs + o] = x;
#pragma unroll
    for (int r = 0; r < kStepCluster; ++r) cluster.map_shared_rank(Xs, r)[(j0 + jj) * Vs + m] = x;
  }
  cluster.sync();
  if (k0 == 0) return;
  // Y1(k0 - NB + j0 + j, m) -= sum_k L(k0 + k, k0 - NB + j0 + j) x(k, m)
#pragma unroll
  for (int f = 0; f < NF; ++f) acc[f][0] = acc[f][1] = 0.0;
  dmma_rows<NF>(Lb + (8 * nf + g) * kSlabLd + 16 * kg + t4, Xs + (16 * kg + t4) * Vs + g, Vs, 4, acc);
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    red[(kg * kStepCols + 8 * nf + g) * (8 * NF) + 8 * f + 2 * t4] = acc[f][0];
    red[(kg * kStepCols + 8 * nf + g) * (8 * NF) + 8 * f + 2 * t4 + 1] = acc[f][1];
  }
  __syncthreads();
  double* y = Y1 + (size_t)(k0 - NB + j0) * Rs;
  for (int o = tid; o < kStepCols * Rs; o += kStepThreads) {
    const int jj = o / Rs, m = o % Rs;
    double d = 0.0;
#pragma unroll
    for (int q = 0; q < kStepKG; ++q) d += red[(q * kStepCols + jj) * (8 * NF) + m];
    y[o] -= d;
  }
}

// Bulk update of the sweep: Y2(n, m) -= sum_k L(k0 + k, n) X_b(k, m) for the columns n < cols of the
// factor's row block b, on the FP64 tensor cores.  A CTA owns 32 columns (one 8-column DMMA
// fragment row per warp); its 128 x 32 tile of L (one 1 KB run per column) and X_b are requested in
// one burst of cp.async, so the kernel pays the memory latency once (the 64 x 64-tile GEMM walks its
// K = 128 in eight dependent slabs: ~20 us per launch whatever the size).
constexpr int kBulkCols = 32, kBulkThreads = 128;
static size_t bulk_smem(int NF) { return (size_t)(kBulkCols * kSlabLd + NB * rhs_stride(NF)) * sizeof(double); }

template <int NF>
__global__ void __launch_bounds__(kBulkThreads)
    k_bwd_bulk(const double* __restrict__ L, long long lda, const double* __restrict__ X, double* __restrict__ Y2,
               int Rs, int k0, int kb, int cols) {
  constexpr int Vs = rhs_stride(NF);
  extern __shared__ __align__(16) double smem[];
  double* Ls = smem;                        // [32][kSlabLd]: Ls[c][k] = L(k0 + k, n0 + c)
  double* Xs = smem + kBulkCols * kSlabLd;  // [NB][Vs]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, n0 = blockIdx.x * kBulkCols;
  const int g = lane >> 2, t4 = lane & 3;
  for (int c = tid; c < kBulkCols * (NB / 2); c += kBulkThreads) {
    const int cc = c / (NB / 2), k = 2 * (c % (NB / 2));
    const bool ok = k < kb && n0 + cc < cols;
    cp_async16(&Ls[cc * kSlabLd + k], ok ? L + (long long)(n0 + cc) * lda + k0 + k : L, ok ? (k + 1 < kb ? 16 : 8) : 0);
  }
  stage_rows(Xs, Vs, X + (size_t)k0 * Rs, Rs, kb, tid, kBulkThreads);
  cp_async_commit();
  for (int c = tid; c < NB * (Vs - Rs); c += kBulkThreads) Xs[(c / (Vs - Rs)) * Vs + Rs + c % (Vs - Rs)] = 0.0;
  cp_async_wait<0>();
  __syncthreads();
  double acc[NF][2];
#pragma unroll
  for (int f = 0; f < NF; ++f) acc[f][0] = acc[f][1] = 0.0;
  dmma_rows<NF>(Ls + (8 * warp + g) * kSlabLd + t4, Xs + t4 * Vs + g, Vs, NB / 4, acc);
  const int nn = n0 + 8 * warp + g;
  if (nn >= cols) return;
  double* y = Y2 + (size_t)nn * Rs;
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    const int m = 8 * f + 2 * t4;  // Rs even: the pair (m, m + 1) is in or out together
    if (m < Rs) {
      double2 v = *reinterpret_cast<double2*>(y + m);
      v.x -= acc[f][0];
      v.y -= acc[f][1];
      *reinterpret_cast<double2*>(y + m) = v;
    }
  }
}

// The whole sweep (one cluster launch and one GEMM per block, joined by events) is
// captured once into a CUDA graph per (matrix, right-hand-side) shape and replayed:
// issued launch by launch it is bound by the host's enqueue rate (~20 us per block for
// two launches, two event records and two waits against ~4 us of device time).
static int enqueue_backward_lookahead(gbem_ctx* ctx, int R, int Rs, double* Y1, double* Y2, double* X, double* d_X,
                                      cudaStream_t s, cudaStream_t chain) {
  const int n = (int)ctx->n;
  const long long lda = ctx->lda;
  const size_t nr = (size_t)n * Rs;
  const int NF = rhs_frags(Rs);
  void (*step)(const double*, const double*, long long, double*, const double*, double*, int, int, int) =
      NF == 1 ? k_bwd_step<1> : NF == 2 ? k_bwd_step<2> : NF == 3 ? k_bwd_step<3> : NF == 4 ? k_bwd_step<4>
      : NF == 6 ? k_bwd_step<6> : k_bwd_step<8>;
  void (*bulk)(const double*, long long, const double*, double*, int, int, int, int) =
      NF == 1 ? k_bwd_bulk<1> : NF == 2 ? k_bwd_bulk<2> : NF == 3 ? k_bwd_bulk<3> : NF == 4 ? k_bwd_bulk<4>
      : NF == 6 ? k_bwd_bulk<6> : k_bwd_bulk<8>;
  const size_t smem = step_smem(NF);
  cudaEvent_t ev_start = ctx->ev_bw[0], ev_step = ctx->ev_bw[1];
  cudaEvent_t* ev_bulk = &ctx->ev_bw[2];  // [3]
  k_border_to_rows<<<(unsigned)((nr + 255) / 256), 256, 0, s>>>(ctx->d_A, lda, n, R, Rs, Y1);
  GBEM_LAUNCH_CHECK(ctx);
  GBEM_CUDA(ctx, cudaMemsetAsync(Y2, 0, nr * sizeof(double), s));
  GBEM_CUDA(ctx, cudaEventRecord(ev_start, s));
  GBEM_CUDA(ctx, cudaStreamWaitEvent(chain, ev_start, 0));
  const double* L = ctx->d_A;
  const int nblk = (n + NB - 1) / NB;
  for (int b = nblk - 1; b >= 0; --b) {
    const int k0 = b * NB, kb = std::min(NB, n - k0);
    if (b + 2 < nblk) GBEM_CUDA(ctx, cudaStreamWaitEvent(chain, ev_bulk[(b + 2) % 3], 0));
    step<<<kStepCluster, kStepThreads, smem, chain>>>(ctx->d_linv + (size_t)b * NB * NB, L, lda, Y1, Y2, X, Rs, k0, kb);
    GBEM_LAUNCH_CHECK(ctx);
    GBEM_CUDA(ctx, cudaEventRecord(ev_step, chain));
    if (b >= 2) {
      GBEM_CUDA(ctx, cudaStreamWaitEvent(s, ev_step, 0));
      const int cols = k0 - NB;  // rows of Y2 above block b - 1
      bulk<<<(unsigned)((cols + kBulkCols - 1) / kBulkCols), kBulkThreads, bulk_smem(NF), s>>>(L, lda, X, Y2, Rs, k0, kb,
                                                                                             cols);
      GBEM_LAUNCH_CHECK(ctx);
      GBEM_CUDA(ctx, cudaEventRecord(ev_bulk[b % 3], s));
    }
  }
  GBEM_CUDA(ctx, cudaStreamWaitEvent(s, ev_step, 0));
  const dim3 tb(32, 8), tg((n + 31) / 32, (R + 31) / 32);
  k_rhs_transpose<<<tg, tb, 0, s>>>(X, n, R, d_X, 0, Rs);
  GBEM_LAUNCH_CHECK(ctx);
  return GBEM_OK;
}

static int solve_backward_lookahead(gbem_ctx* ctx, int R, double* d_X) {
  const int n = (int)ctx->n;
  const int Rs = (R + 1) & ~1;
  cudaStream_t s = ctx->stream, chain = ctx->side_stream;
  const size_t nr = (size_t)n * Rs;
  if (ctx->sw_cap < 3 * nr) {
    cudaFree(ctx->d_sw);
    ctx->d_sw = nullptr;
    ctx->sw_cap = 0;
    GBEM_CUDA(ctx, cudaMalloc(&ctx->d_sw, 3 * nr * sizeof(double)));
    ctx->sw_cap = 3 * nr;
  }
  double* Y1 = ctx->d_sw;
  double* Y2 = Y1 + nr;
  double* X = Y2 + nr;
  if (!(ctx->attr_set & gbem_ctx::kAttrBwdStep)) {
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_bwd_step<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)step_smem(1)));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_bwd_step<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)step_smem(2)));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_bwd_step<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)step_smem(3)));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_bwd_step<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)step_smem(4)));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_bwd_step<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)step_smem(6)));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_bwd_step<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)step_smem(8)));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_bwd_bulk<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bulk_smem(1)));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_bwd_bulk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bulk_smem(2)));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_bwd_bulk<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bulk_smem(3)));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_bwd_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bulk_smem(4)));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_bwd_bulk<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bulk_smem(6)));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_bwd_bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bulk_smem(8)));
    ctx->attr_set |= gbem_ctx::kAttrBwdStep;
  }
  for (auto& e : ctx->ev_bw)
    if (!e) GBEM_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  static const bool no_graph = getenv("GBEM_NO_BWD_GRAPH") != nullptr;
  // (the legacy default stream cannot be captured: issue the launches directly)
  if (no_graph || s == nullptr || s == cudaStreamLegacy)
    return enqueue_backward_lookahead(ctx, R, Rs, Y1, Y2, X, d_X, s, chain);
  // graph cache: one instantiated sweep per (shape, buffers)
  gbem_ctx::BwdGraphKey key{ctx->d_A, ctx->d_linv, Y1, d_X, ctx->lda, n, R};
  if (!ctx->bw_graph_exec || !(ctx->bw_graph_key == key)) {
    if (ctx->bw_graph_exec) {
      cudaGraphExecDestroy((cudaGraphExec_t)ctx->bw_graph_exec);
      ctx->bw_graph_exec = nullptr;
    }
    const int64_t launches0 = ctx->launches;
    GBEM_CUDA(ctx, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    int rc = enqueue_backward_lookahead(ctx, R, Rs, Y1, Y2, X, d_X, s, chain);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(s, &graph);
    ctx->launches = launches0;
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (e != cudaSuccess) return ctx->fail(GBEM_ECUDA, std::string("backward-sweep graph capture: ") + cudaGetErrorString(e));
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return ctx->fail(GBEM_ECUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
    ctx->bw_graph_exec = exec;
    ctx->bw_graph_key = key;
    ctx->bw_graph_launches = 2 * ((n + NB - 1) / NB);  // kernels per replay: nblk steps, nblk - 2 bulk GEMMs, 2 copies
  }
  GBEM_CUDA(ctx, cudaGraphLaunch((cudaGraphExec_t)ctx->bw_graph_exec, s));
  ctx->launches += ctx->bw_graph_launches;
  return GBEM_OK;
}

namespace {

int ensure_work(gbem_ctx* ctx, size_t elems) {
  if (ctx->work_cap >= elems && ctx->d_work) return GBEM_OK;
  if (ctx->d_work) cudaFree(ctx->d_work);
  ctx->d_work = nullptr;
  ctx->work_cap = 0;
  GBEM_CUDA(ctx, cudaMalloc(&ctx->d_work, elems * sizeof(double)));
  ctx->work_cap = elems;
  return GBEM_OK;
}

}  // namespace

// SM partition for the factorisation (green contexts, driver API reached
// through the runtime's entry-point query: no link-time libcuda dependency).
// GBEM_GREEN_SIDE = SMs reserved for the diagonal-block factor (default 2).
static int init_green(gbem_ctx* ctx) {
  if (ctx->green_state) return ctx->green_state;
  ctx->green_state = -1;
  PFN_cuDeviceGet p_get = nullptr;
  PFN_cuDeviceGetDevResource p_res = nullptr;
  PFN_cuDevSmResourceSplitByCount p_split = nullptr;
  PFN_cuDevResourceGenerateDesc p_desc = nullptr;
  PFN_cuGreenCtxCreate p_create = nullptr;
  PFN_cuGreenCtxStreamCreate p_stream = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuDeviceGet", (void**)&p_get, cudaEnableDefault, &q) != cudaSuccess || !p_get ||
      cudaGetDriverEntryPoint("cuDeviceGetDevResource", (void**)&p_res, cudaEnableDefault, &q) != cudaSuccess || !p_res ||
      cudaGetDriverEntryPoint("cuDevSmResourceSplitByCount", (void**)&p_split, cudaEnableDefault, &q) != cudaSuccess ||
      !p_split ||
      cudaGetDriverEntryPoint("cuDevResourceGenerateDesc", (void**)&p_desc, cudaEnableDefault, &q) != cudaSuccess ||
      !p_desc || cudaGetDriverEntryPoint("cuGreenCtxCreate", (void**)&p_create, cudaEnableDefault, &q) != cudaSuccess ||
      !p_create ||
      cudaGetDriverEntryPoint("cuGreenCtxStreamCreate", (void**)&p_stream, cudaEnableDefault, &q) != cudaSuccess ||
      !p_stream) {
    cudaGetLastError();
    return ctx->green_state;
  }
  CUdevice dev;
  if (p_get(&dev, ctx->device) != CUDA_SUCCESS) return ctx->green_state;
  CUdevResource all, side, rest;
  if (p_res(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return ctx->green_state;
  const int want = getenv("GBEM_GREEN_SIDE") ? atoi(getenv("GBEM_GREEN_SIDE")) : 2;
  unsigned ng = 1;
  // CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING: without it a request for 2 SMs reserves 8 on
  // sm_100 (tools/green_probe.cu: side 8 / rest 140), and the trailing updates lose 6 SMs = 4% of
  // the machine; with it the split is 2 / 146.  No kernel of either partition uses clusters.
  const unsigned split_flags = getenv("GBEM_GREEN_FLAGS") ? (unsigned)atoi(getenv("GBEM_GREEN_FLAGS"))
                                                          : (unsigned)CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING;
  if (p_split(&side, &ng, &all, &rest, split_flags, (unsigned)want) != CUDA_SUCCESS || ng != 1) return ctx->green_state;
  CUdevResourceDesc d_side, d_rest;
  if (p_desc(&d_side, &side, 1) != CUDA_SUCCESS || p_desc(&d_rest, &rest, 1) != CUDA_SUCCESS) return ctx->green_state;
  CUgreenCtx g_side, g_main;
  if (p_create(&g_side, d_side, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) return ctx->green_state;
  if (p_create(&g_main, d_rest, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) return ctx->green_state;
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  CUstream ss, sm;
  if (p_stream(&ss, g_side, CU_STREAM_NON_BLOCKING, hi) != CUDA_SUCCESS) return ctx->green_state;
  if (p_stream(&sm, g_main, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) return ctx->green_state;
  CUstream sh;
  if (p_stream(&sh, g_main, CU_STREAM_NON_BLOCKING, hi) != CUDA_SUCCESS) return ctx->green_state;
  CUstream sl;
  if (p_stream(&sl, g_side, CU_STREAM_NON_BLOCKING, lo) != CUDA_SUCCESS) return ctx->green_state;
  ctx->g_side = (cudaStream_t)ss;
  ctx->g_side_lo = (cudaStream_t)sl;
  ctx->g_main = (cudaStream_t)sm;
  ctx->g_main_hi = (cudaStream_t)sh;
  ctx->green_ctx[0] = (void*)g_side;
  ctx->green_ctx[1] = (void*)g_main;
  ctx->green_side_sms = (int)side.sm.smCount;
  if (cudaEventCreateWithFlags(&ctx->ev_gs, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_ge, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_gt, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_gra, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_side_pre, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_side_done, cudaEventDisableTiming) != cudaSuccess)
    return ctx->green_state;
  ctx->green_state = 1;
  return ctx->green_state;
}

// Blocked Cholesky of ctx->d_A (n x n) + solves for nrhs columns of d_B (ld n)
// into d_X; d_resid[nrhs] optional.
// Blocked Cholesky of ctx->d_A in place (lower triangle <- L, diagonal saved,
// strict upper triangle untouched); inverses of the diagonal blocks kept in
// ctx->d_linv.  Non-SPD: GBEM_ENUMERIC "matrix not positive definite (pivot at row k)".
int gbem_internal_factor(gbem_ctx* ctx, gbem_solve_stats* stats) {
  const int n = (int)ctx->n;
  const long long lda = ctx->lda;
  if (stats) {
    *stats = gbem_solve_stats{};
    stats->n = n;
    stats->bad_pivot = -1;
  }
  if (n == 0) return GBEM_OK;
  if (ctx->factored) return ctx->fail(GBEM_EINVAL, "matrix already factored; re-assemble or re-upload");
  const int nblk = (n + NB - 1) / NB;
  // inverses of the diagonal blocks, kept with the factor for the solves
  const size_t need_linv = (size_t)nblk * NB * NB;
  if (ctx->linv_cap < need_linv) {
    cudaFree(ctx->d_linv);
    ctx->d_linv = nullptr;
    ctx->linv_cap = 0;
    GBEM_CUDA(ctx, cudaMalloc(&ctx->d_linv, need_linv * sizeof(double)));
    ctx->linv_cap = need_linv;
  }
  double* Linv = ctx->d_linv;
  if (ctx->diag_cap < n) {
    if (ctx->d_diag) cudaFree(ctx->d_diag);
    GBEM_CUDA(ctx, cudaMalloc(&ctx->d_diag, sizeof(double) * n));
    ctx->diag_cap = n;
  }
  if (!ctx->d_info) {
    GBEM_CUDA(ctx, cudaMalloc(&ctx->d_info, sizeof(int)));
    GBEM_CUDA(ctx, cudaMallocHost(&ctx->h_info, sizeof(int)));
  }
  if (!(ctx->attr_set & gbem_ctx::kAttrFactor)) {
    GBEM_CUDA(ctx, cudaFuncSetAttribute(kUpdate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kUpdSmemPadded));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(kUpdateBulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kUpdSmemPadded));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_trsm_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTrsmSmem));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_potrf_diag, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kPotrfSmem));
    ctx->attr_set |= gbem_ctx::kAttrFactor;
  }
  cudaStream_t s = ctx->stream;
  int big = 0x7fffffff;
  GBEM_CUDA(ctx, cudaMemcpyAsync(ctx->d_info, &big, sizeof(int), cudaMemcpyHostToDevice, s));
  k_save_diag<<<(n + 255) / 256, 256, 0, s>>>(ctx->d_A, lda, n, ctx->d_diag);
  GBEM_LAUNCH_CHECK(ctx);
  cudaEventRecord(ctx->ev[0], s);
  // Look-ahead: the diagonal factor + panel trsm of block k+1 run on the
  // high-priority side stream while the main stream finishes the trailing
  // update of block k (only block column k+1 has to be updated first).
  if (!ctx->side_stream) {
    int lo = 0, hi = 0;
    GBEM_CUDA(ctx, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    GBEM_CUDA(ctx, cudaStreamCreateWithPriority(&ctx->side_stream, cudaStreamNonBlocking, hi));
    GBEM_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_panel, cudaEventDisableTiming));
    GBEM_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_col, cudaEventDisableTiming));
  }
  cudaStream_t s_side = ctx->side_stream;
  static const int tail_rows = getenv("GBEM_FACTOR_TAIL") ? atoi(getenv("GBEM_FACTOR_TAIL")) : 1024;
  GBEM_CUDA(ctx, cudaEventRecord(ctx->ev_col, s));
  // GBEM_FACTOR_PROFILE=1: per-block side-stream (diagonal factor + panel trsm)
  // and main-stream timings on stderr (diagnostics only)
  static const bool prof = getenv("GBEM_FACTOR_PROFILE") != nullptr;
  std::vector<cudaEvent_t> pe;
  std::vector<int> sb_starts;  // first block of every pipelined super-block (profile mode)
  if (prof) {
    pe.resize(6 * (size_t)nblk);
    for (auto& e : pe) cudaEventCreate(&e);
  }
  static const bool no_green = getenv("GBEM_NO_GREEN") != nullptr;
  const bool green = !no_green && n >= 2 * tail_rows && init_green(ctx) == 1;
  if (green) {
    // Look-ahead on an SM partition.  U(b, c) = update of block column c by
    // L21 of block b.  Three streams:
    //   p  (reserved SMs)           potrf(b+1)
    //   hi (main SMs, high prio.)   trsm(b+1), band(b+1) = U(b+1, b+2)
    //   lo (main SMs)               rest_a(b) = U(b, b+2), rest_b(b) = U(b, >= b+3)
    // so the latency-bound chain potrf -> trsm -> band of the next blocks runs
    // under the bulk trailing update; rest_a splits off the column that the
    // next band update writes (no two updates of one column run concurrently).
    // Events: P (potrf done), T (trsm done), B (band done), RA (rest_a done).
    cudaStream_t lo = ctx->g_main, hi = ctx->g_main_hi, p = ctx->g_side;
    cudaEvent_t evP = ctx->ev_panel, evB = ctx->ev_col, evT = ctx->ev_gt;
    if (!ctx->d_band_done) GBEM_CUDA(ctx, cudaMalloc(&ctx->d_band_done, sizeof(unsigned)));
    GBEM_CUDA(ctx, cudaMemsetAsync(ctx->d_band_done, 0, sizeof(unsigned), s));
    GBEM_CUDA(ctx, cudaEventRecord(ctx->ev_gs, s));
    GBEM_CUDA(ctx, cudaStreamWaitEvent(lo, ctx->ev_gs, 0));
    GBEM_CUDA(ctx, cudaStreamWaitEvent(hi, ctx->ev_gs, 0));
    GBEM_CUDA(ctx, cudaStreamWaitEvent(p, ctx->ev_gs, 0));
    constexpr int kBand = NB / 64;  // tile columns per block column
    static const int fdbg = getenv("GBEM_FACTOR_DBG") ? atoi(getenv("GBEM_FACTOR_DBG")) : 0;  // timing experiments (results wrong)
    auto trailing = [&](int b, int& m, int& nt, double*& A21, double*& A22) {
      const int k0 = b * NB, kb = std::min(NB, n - k0);
      m = n - k0 - kb + (int)ctx->border;
      nt = (m + 63) / 64;
      A21 = ctx->d_A + (long long)k0 * lda + k0 + kb;
      A22 = ctx->d_A + (long long)(k0 + kb) * lda + (k0 + kb);
    };
    auto potrf = [&](int b, cudaStream_t st, unsigned wait_target = 0) {
      const int k0 = b * NB, kb = std::min(NB, n - k0);
      k_potrf_diag<<<1, kPotrfThreads, kPotrfSmem, st>>>(ctx->d_A + (long long)k0 * lda + k0, lda, kb, k0,
                                                         Linv + (size_t)b * NB * NB, ctx->d_info,
                                                         wait_target ? ctx->d_band_done : nullptr, wait_target);
    };
    auto trsm = [&](int b, cudaStream_t st) {
      int m, nt;
      double *A21, *A22;
      trailing(b, m, nt, A21, A22);
      const int kb = std::min(NB, n - b * NB);
      if (m > 0 && !(fdbg & 1))
        k_trsm_rows<<<(unsigned)((m + kTrsmRows - 1) / kTrsmRows), kTrsmThreads, kTrsmSmem, st>>>(
            A21, lda, A21, lda, Linv + (size_t)b * NB * NB, NB, m, kb, kb);
    };
    // U(b, b+1+j) for j = j0 (one block column; tile columns [kBand j0, kBand j0 + kBand))
    auto update_col = [&](int b, int j0, cudaStream_t st) {
      int m, nt;
      double *A21, *A22;
      trailing(b, m, nt, A21, A22);
      const int t0 = kBand * j0;
      if (t0 >= nt) return;
      launch_update(ctx, dim3(nt, std::min(kBand, nt - t0)), false, st, A22, lda, A21, lda, m, std::min(NB, n - b * NB),
                    t0, std::min(kBand, nt - t0));
    };
    // U(b, >= b+1+j0)
    auto update_from = [&](int b, int j0, cudaStream_t st) {
      int m, nt;
      double *A21, *A22;
      trailing(b, m, nt, A21, A22);
      const int t0 = kBand * j0;
      if (t0 >= nt) return;
      const long long tiles = (long long)(nt - t0) * (nt - t0 + 1) / 2;
      launch_update(ctx, dim3((unsigned)tiles), false, st, A22, lda, A21, lda, m, std::min(NB, n - b * NB), t0, 0);
    };
    // Super-blocks of two 128-column blocks: the diagonal factors and panel
    // trsms stay at 128 columns (chain on p / hi), the trailing update of a
    // super-block is one K = 256 DMMA update (band2: the next super-block's
    // columns, then rest2: everything right of it), which amortises each
    // tile's C read-modify-write over twice the flops of a K = 128 update.
    //   p/hi: stepA(s+1) = potrf, trsm, U(b, b+1), potrf, trsm   (after band2(s))
    //   lo:   band2(s) -> rest2(s) -> [T(s+1)] band2(s+1) -> ...
    // U(., c) for one column never runs concurrently on two streams.
    // wait_target > 0: the first diagonal factor waits on the band counter
    // (combined band + rest update on lo) instead of an event after the band
    auto stepA = [&](int b0, int nb, unsigned wait_target) -> int {
      if (!wait_target) GBEM_CUDA(ctx, cudaStreamWaitEvent(p, evB, 0));
      for (int k = 0; k < nb; ++k) {
        const int bb = b0 + k;
        if (k > 0) {
          // U(b0 .. b0+k-1, b0 + k): block column b0 + k by the super-block's
          // first k blocks at once (one K = 128 k update on the chain)
          const int c0 = bb * NB, mk = n - c0 + (int)ctx->border, ntk = (mk + 63) / 64;
          if (!(fdbg & 2))
            launch_update(ctx, dim3(ntk, std::min(kBand, ntk)), false, hi, ctx->d_A + (long long)c0 * lda + c0, lda,
                          ctx->d_A + (long long)(b0 * NB) * lda + c0, lda, mk, k * NB, 0, std::min(kBand, ntk));
          GBEM_LAUNCH_CHECK(ctx);
          GBEM_CUDA(ctx, cudaEventRecord(evB, hi));
          GBEM_CUDA(ctx, cudaStreamWaitEvent(p, evB, 0));
        }
        if (prof) cudaEventRecord(pe[6 * bb], p);
        potrf(bb, p, k == 0 ? wait_target : 0u);
        GBEM_LAUNCH_CHECK(ctx);
        if (prof) cudaEventRecord(pe[6 * bb + 1], p);
        GBEM_CUDA(ctx, cudaEventRecord(evP, p));
        GBEM_CUDA(ctx, cudaStreamWaitEvent(hi, evP, 0));
        trsm(bb, hi);
        GBEM_LAUNCH_CHECK(ctx);
        if (prof) cudaEventRecord(pe[6 * bb + 2], hi);
      }
      GBEM_CUDA(ctx, cudaEventRecord(evT, hi));
      return GBEM_OK;
    };
    // U([b0, b0 + nb), block columns >= b0 + nb + j0): band (j0 = 0, one super-
    // block of kBand2 tile columns) or triangular rest (j0 = 2)
    // super-block width in 128-column blocks (K of the trailing update = SB * 128;
    // tools/gemm_bench.cu at m = 20,000: K = 256 / 384 / 512 / 640 -> 32.0 / 33.0 / 33.4 / 33.8 TFLOP/s).
    // The intra-super-block updates lengthen the potrf / trsm chain by O(SB^2)
    // thin updates, which a small trailing matrix cannot hide.
    static const int sb_env = getenv("GBEM_SUPERBLOCK") ? std::max(1, atoi(getenv("GBEM_SUPERBLOCK"))) : 0;
    // Adaptive width: wide super-blocks while the trailing matrix is large (the update amortises
    // its C read-modify-write over K = 128 SB and hides the O(SB^2) chain), narrower ones as it
    // shrinks and the chain (SB diagonal factors of ~47 us, SB trsms, the intra-super-block
    // updates) would outlast the update.  GBEM_SB_SCHED="sb:rows,..." overrides the table
    // (first entry whose rows <= remaining rows), GBEM_SUPERBLOCK=k fixes the width.
    struct SbRule { int sb, rows; };
    static const std::vector<SbRule> sb_env_rules = [] {
      std::vector<SbRule> r;
      if (const char* e = getenv("GBEM_SB_SCHED")) {
        int sb = 0, rows = 0, used = 0;
        while (sscanf(e, "%d:%d%n", &sb, &rows, &used) == 2) {
          r.push_back({std::max(1, sb), rows});
          e += used;
          if (*e == ',') ++e;
        }
      }
      return r;
    }();
    // config 3: 411.1 ms at a fixed SB = 5, 405.5 at 10, 403.3 with the large table;
    // config 2: 18.47 ms at a fixed SB = 2, 18.23 with the small one (bulk-staged update: 17.49 with
    // {4, 3, 2, 1}, 17.34 with {6, 4, 2, 1})
    static const std::vector<SbRule> sb_large = {{12, 16000}, {10, 12000}, {8, 9000}, {6, 7000},
                                                 {4, 5000},   {3, 3500},   {2, 0}};
    static const std::vector<SbRule> sb_small = {{6, 9000}, {4, 6000}, {2, 3000}, {1, 0}};
    static const bool ramp_on = getenv("GBEM_SB_NO_RAMP") == nullptr;
    static const std::vector<int> ramp_widths = [] {
      std::vector<int> w;
      if (const char* e = getenv("GBEM_SB_RAMP")) {
        int v = 0, used = 0;
        while (sscanf(e, "%d%n", &v, &used) == 1) {
          w.push_back(std::max(1, v));
          e += used;
          if (*e == ',') ++e;
        }
      }
      return w;
    }();
    static const bool ramp_env = getenv("GBEM_SB_RAMP") != nullptr;
    static const std::vector<int> ramp_small = {2}, ramp_large = {4, 8};
    auto sb_at = [&](int blk) {
      if (sb_env > 0) return sb_env;
      const int rows = n - blk * NB;
      // ramp: nothing overlaps the first super-block's chain (12 diagonal factors, trsms and
      // intra-super-block updates at full height: 3.6 ms), so the first ones are narrower
      // (worth 0.1 ms on config 2; on config 3 the early K = 512 / 1,024 updates give it back)
      int ramp = 1 << 20;
      if (ramp_on) {
        int at = 0;
        for (int w : ramp_env ? ramp_widths : (n < 16384 ? ramp_small : ramp_large)) {
          if (blk == at) ramp = w;
          at += w;
        }
      }
      for (const SbRule& r : !sb_env_rules.empty() ? sb_env_rules : (n < 16384 ? sb_small : sb_large))
        if (rows >= r.rows) return std::min(r.sb, ramp);
      return 1;
    };
    static const int occ_rows = getenv("GBEM_OCC_ROWS") ? atoi(getenv("GBEM_OCC_ROWS")) : 0;
    static const bool combined = getenv("GBEM_NO_COMBINED") == nullptr;
    auto update2 = [&](int b0, int nb, bool band_part, int kBand2) {
      const int k0 = b0 * NB, kw = std::min(nb * NB, n - k0);
      const int m = n - k0 - kw + (int)ctx->border;
      if (m <= 0) return;
      const int nt = (m + 63) / 64;
      double* A21 = ctx->d_A + (long long)k0 * lda + k0 + kw;
      double* A22 = ctx->d_A + (long long)(k0 + kw) * lda + (k0 + kw);
      if (band_part) {
        launch_update(ctx, dim3(nt, std::min(kBand2, nt)), false, lo, A22, lda, A21, lda, m, kw, 0,
                      std::min(kBand2, nt));
      } else if (nt > kBand2) {
        const long long tiles = (long long)(nt - kBand2) * (nt - kBand2 + 1) / 2;
        // near the end the chain on p / hi is the critical path: the rest update
        // then runs 3 CTAs per SM (padded shared memory), which keeps one slot
        // per SM free for the chain's trsm / band kernels instead of queueing
        // them behind a full wave of update tiles
        launch_update(ctx, dim3((unsigned)tiles), m < occ_rows, lo, A22, lda, A21, lda, m, kw, kBand2, 0);
      }
    };
    GBEM_CUDA(ctx, cudaEventRecord(evB, p));  // stepA(0) waits on nothing
    int b = 0;
    int rc2 = stepA(0, std::min(sb_at(0), nblk), 0u);
    if (rc2) return rc2;
    unsigned band_target = 0;  // cumulative band CTAs of the combined updates
    for (;;) {
      const int nb = std::min(sb_at(b), nblk - b), next = b + nb;
      // the band of this update = the next super-block's columns
      const int nb_next = next < nblk ? std::min(sb_at(next), nblk - next) : 1;
      const int kBand2 = nb_next * kBand;
      if (prof) {
        cudaEventRecord(pe[6 * b + 3], lo);  // previous update done: lo idle until the chain's trsm (evT)
        sb_starts.push_back(b);
      }
      GBEM_CUDA(ctx, cudaStreamWaitEvent(lo, evT, 0));
      if (prof) cudaEventRecord(pe[6 * b + 5], lo);
      if (next >= nblk) {  // the last super-block: its trsm covered the border rows
        update2(b, nb, true, kBand2);
        GBEM_LAUNCH_CHECK(ctx);
        b = nblk;
        break;
      }
      const bool next_tail = n - next * NB < tail_rows;
      if (combined) {
        // band2(b) and rest2(b) in one launch, band tiles first; stepA(next)
        // starts on the band counter, so the chain does not wait for the
        // band launch's partial last wave and rest2 fills the machine at once
        const int k0 = b * NB, kw = std::min(nb * NB, n - k0);
        const int m = n - k0 - kw + (int)ctx->border, nt = (m + 63) / 64;
        const int bw = std::min(kBand2, nt);
        const long long tiles =
            (long long)nt * bw + (nt > kBand2 ? (long long)(nt - kBand2) * (nt - kBand2 + 1) / 2 : 0);
        double* A21 = ctx->d_A + (long long)k0 * lda + k0 + kw;
        double* A22 = ctx->d_A + (long long)(k0 + kw) * lda + (k0 + kw);
        // Experiment (off by default, GBEM_SIDE_SHARE=fraction): the 2 SMs reserved for the diagonal
        // factor idle most of the time, so while the update is long against the chain (m >= 12,000,
        // K >= 1,024) the last `side_share` of its tiles (far from the band) can run on them at low
        // priority.  Measured on config 3: 0.006 -> factor 371.2 -> 369.6 ms, 0.009 -> 380.5 ms,
        // 0.012 -> 500 ms: the diagonal factor does not get ahead of the share's queued CTAs, so as
        // soon as the share outlasts the chain's slack the chain becomes the critical path.
        static const double side_share = getenv("GBEM_SIDE_SHARE") ? atof(getenv("GBEM_SIDE_SHARE")) : 0.0;
        long long t_side = 0;
        if (side_share > 0 && ctx->g_side_lo && m >= 12000 && kw >= 1024 && kw % 16 == 0 && lda % 2 == 0 &&
            ((m & 1) == 0 || k0 + kw + m < lda) && getenv("GBEM_UPDATE_CPASYNC") == nullptr)
          t_side = std::min<long long>((long long)(side_share * (double)tiles), tiles - (long long)nt * bw - 1);
        if (t_side > 0) {
          GBEM_CUDA(ctx, cudaEventRecord(ctx->ev_side_pre, lo));  // after evT and the previous update
          GBEM_CUDA(ctx, cudaStreamWaitEvent(ctx->g_side_lo, ctx->ev_side_pre, 0));
          kUpdateBulk<<<(unsigned)t_side, BulkUpd::THREADS, BulkUpd::SMEM, ctx->g_side_lo>>>(
              A22, lda, A21, lda, m, kw, 0, -bw, ctx->d_band_done, tiles - t_side);
          GBEM_LAUNCH_CHECK(ctx);
          GBEM_CUDA(ctx, cudaEventRecord(ctx->ev_side_done, ctx->g_side_lo));
        } else {
          t_side = 0;
        }
        launch_update(ctx, dim3((unsigned)(tiles - t_side)), false, lo, A22, lda, A21, lda, m, kw, 0, -bw,
                      ctx->d_band_done);
        GBEM_LAUNCH_CHECK(ctx);
        if (t_side > 0) GBEM_CUDA(ctx, cudaStreamWaitEvent(lo, ctx->ev_side_done, 0));
        band_target += (unsigned)(nt * bw);
        if (!next_tail) {
          rc2 = stepA(next, nb_next, band_target);
          if (rc2) return rc2;
        }
      } else {
        update2(b, nb, true, kBand2);  // band2(b): the next super-block's columns
        GBEM_LAUNCH_CHECK(ctx);
        GBEM_CUDA(ctx, cudaEventRecord(evB, lo));
        if (!next_tail) {
          rc2 = stepA(next, nb_next, 0u);
          if (rc2) return rc2;
        }
        update2(b, nb, false, kBand2);  // rest2(b)
        GBEM_LAUNCH_CHECK(ctx);
      }
      if (prof) cudaEventRecord(pe[6 * b + 4], lo);
      b = next;
      if (next_tail) break;
    }
    // tail: one stream, in order (the band update of the last pipelined block
    // and everything on hi are joined first)
    GBEM_CUDA(ctx, cudaStreamWaitEvent(lo, evB, 0));
    for (; b < nblk; ++b) {
      potrf(b, lo);
      GBEM_LAUNCH_CHECK(ctx);
      trsm(b, lo);
      GBEM_LAUNCH_CHECK(ctx);
      update_from(b, 0, lo);
      GBEM_LAUNCH_CHECK(ctx);
    }
    GBEM_CUDA(ctx, cudaEventRecord(ctx->ev_ge, lo));
    GBEM_CUDA(ctx, cudaStreamWaitEvent(s, ctx->ev_ge, 0));
  }
  for (int b = 0; b < (green ? 0 : nblk); ++b) {
    int k0 = b * NB, kb = std::min(NB, n - k0);
    // rows below the diagonal block: the remaining matrix rows plus the border
    // rows of a bordered factorisation (ctx->border, gbem_ctx.cuh)
    int m = n - k0 - kb + (int)ctx->border;
    double* Akk = ctx->d_A + (long long)k0 * lda + k0;
    double* A21 = Akk + kb;  // rows k0+kb.., cols k0..
    // tail: once the trailing matrix is small the look-ahead has nothing to
    // overlap, and the cross-stream event hops only add latency to the chain
    const bool tail = n - k0 < tail_rows;
    cudaStream_t s1 = tail ? s : s_side;
    if (!tail) GBEM_CUDA(ctx, cudaStreamWaitEvent(s1, ctx->ev_col, 0));
    if (prof) cudaEventRecord(pe[6 * b], s1);
    k_potrf_diag<<<1, kPotrfThreads, kPotrfSmem, s1>>>(Akk, lda, kb, k0, Linv + (size_t)b * NB * NB, ctx->d_info);
    GBEM_LAUNCH_CHECK(ctx);
    if (m > 0) {
      // L21 = A21 * inv(L11)^T  (in place, one CTA per 32-row strip)
      k_trsm_rows<<<(unsigned)((m + kTrsmRows - 1) / kTrsmRows), kTrsmThreads, kTrsmSmem, s1>>>(
          A21, lda, A21, lda, Linv + (size_t)b * NB * NB, NB, m, kb, kb);
      GBEM_LAUNCH_CHECK(ctx);
    }
    if (prof) cudaEventRecord(pe[6 * b + 1], s1);
    if (!tail) {
      GBEM_CUDA(ctx, cudaEventRecord(ctx->ev_panel, s1));
      GBEM_CUDA(ctx, cudaStreamWaitEvent(s, ctx->ev_panel, 0));
    }
    if (prof) cudaEventRecord(pe[6 * b + 2], s);
    if (m <= 0) break;
    // A22 -= L21 L21^T on 64 x 64 lower tiles: first the next block column
    // (kBand tile columns), then the rest
    const int nt = (m + 63) / 64;
    double* A22 = ctx->d_A + (long long)(k0 + kb) * lda + (k0 + kb);
    constexpr int kBand = NB / 64;
    const int band = std::min(kBand, nt);
    launch_update(ctx, dim3(nt, band), false, s, A22, lda, A21, lda, m, kb, 0, band);
    GBEM_LAUNCH_CHECK(ctx);
    GBEM_CUDA(ctx, cudaEventRecord(ctx->ev_col, s));
    if (prof) cudaEventRecord(pe[6 * b + 3], s);
    if (nt > kBand) {
      const long long rest = (long long)(nt - kBand) * (nt - kBand + 1) / 2;
      launch_update(ctx, dim3((unsigned)rest), false, s, A22, lda, A21, lda, m, kb, kBand, 0);
      GBEM_LAUNCH_CHECK(ctx);
    }
  }
  cudaEventRecord(ctx->ev[1], s);
  GBEM_CUDA(ctx, cudaMemcpyAsync(ctx->h_info, ctx->d_info, sizeof(int), cudaMemcpyDeviceToHost, s));
  if (ctx->async && !stats && !prof) {
    // stream-ordered mode: the pivot check is deferred to gbem_ctx_sync
    ctx->factored = true;
    ctx->info_pending = true;
    return GBEM_OK;
  }
  GBEM_CUDA(ctx, cudaStreamSynchronize(s));
  if (prof) {
    double side = 0, band = 0, gap = 0;
    for (int b = 0; b < nblk; ++b) {
      float x = 0;
      if (cudaEventElapsedTime(&x, pe[6 * b], pe[6 * b + 1]) == cudaSuccess) side += x;
      if (b + 1 < nblk && cudaEventElapsedTime(&x, pe[6 * b + 2], pe[6 * b + 3]) == cudaSuccess) band += x;
      if (b > 0 && cudaEventElapsedTime(&x, pe[6 * (b - 1) + 3], pe[6 * b]) == cudaSuccess) gap += x;
    }
    cudaGetLastError();
    fprintf(stderr, "[factor profile] n=%d blocks=%d mode=%s (SM partition %d + %d) side=%.3f ms band-update=%.3f ms "
            "band->next-potrf gap=%.3f ms\n", n, nblk, green ? "green" : "streams", green ? ctx->green_side_sms : 0,
            green ? ctx->num_sms - ctx->green_side_sms : ctx->num_sms, side, band, gap);
    if (green) {
      // per super-block on lo (us): idle wait for the chain's last trsm, then the combined
      // band + rest update; potrf includes its spin on the band counter
      double tw = 0, tu = 0, tfl = 0;
      for (size_t k = 0; k < sb_starts.size(); ++k) {
        const int b = sb_starts[k];
        float w = 0, u = 0;
        cudaEventElapsedTime(&w, pe[6 * b + 3], pe[6 * b + 5]);
        if (cudaEventElapsedTime(&u, pe[6 * b + 5], pe[6 * b + 4]) != cudaSuccess) u = 0;
        cudaGetLastError();
        const int k0 = b * NB, kw = std::min((int)NB * (k + 1 < sb_starts.size() ? sb_starts[k + 1] - b : nblk - b), n - k0);
        const double m = n - k0 - kw + (double)ctx->border;
        const double fl = m * (m + 1) * kw;  // lower triangle, 2 flops per entry and k
        tw += w; tu += u; tfl += u > 0 ? fl : 0;
        if (k % 4 == 0 || k + 8 >= sb_starts.size())
          fprintf(stderr, "  sb %3d (blk %3d, m %6.0f, K %4d): lo idle %7.1f us, update %8.1f us = %5.2f TFLOP/s\n", (int)k, b,
                  m, kw, 1e3 * w, 1e3 * u, u > 0 ? fl / (u * 1e-3) * 1e-12 : 0.0);
      }
      fprintf(stderr, "  totals: lo idle %.3f ms, updates %.3f ms (%.2f TFLOP/s while running)\n", tw, tu,
              tu > 0 ? tfl / (tu * 1e-3) * 1e-12 : 0.0);
    }
    for (auto& e : pe) cudaEventDestroy(e);
  }
  ctx->factored = true;
  if (*ctx->h_info != big) {
    if (stats) stats->bad_pivot = *ctx->h_info;
    return ctx->fail(GBEM_ENUMERIC,
                     "matrix not positive definite (pivot at row " + std::to_string(*ctx->h_info) + ")");
  }
  if (stats) {
    float a = 0;
    cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]);
    stats->ms_factor = a;
  }
  return GBEM_OK;
}

// Y = A X (n x R each, column-major) with the symmetric matrix given by the
// preserved strict upper triangle and the saved diagonal: valid before and
// after the factorisation (the residual of solver.hpp:47, gbem_matrix_apply_dev).
static int apply_sym(gbem_ctx* ctx, const double* X, int R, double* Y) {
  const int n = (int)ctx->n;
  const long long lda = ctx->lda;
  cudaStream_t s = ctx->stream;
    // A X on the tensor cores, one pass over A per 32 right-hand sides
    // (k_symm_dmma: config 3 6.2 -> 2.6 ms); below n = 16,384 its 64-row CTAs
    // cannot fill the machine and the scalar k_symv_upper (column chunks) is
    // faster (config 2: 0.27 vs 0.55 ms).  GBEM_SYMV_SCALAR=1 forces the scalar one.
    static const bool force_scalar = getenv("GBEM_SYMV_SCALAR") != nullptr;
    const bool scalar = force_scalar || n < 16384;
    if (!scalar) {
      if (!(ctx->attr_set & gbem_ctx::kAttrSymm)) {
        GBEM_CUDA(ctx, cudaFuncSetAttribute(k_symm_dmma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)SymmShape<8>::SMEM));
        GBEM_CUDA(ctx, cudaFuncSetAttribute(k_symm_dmma<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)SymmShape<16>::SMEM));
        GBEM_CUDA(ctx, cudaFuncSetAttribute(k_symm_dmma<24>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)SymmShape<24>::SMEM));
        GBEM_CUDA(ctx, cudaFuncSetAttribute(k_symm_dmma<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)SymmShape<32>::SMEM));
        ctx->attr_set |= gbem_ctx::kAttrSymm;
      }
      const unsigned grid = (unsigned)((n + kSyT - 1) / kSyT);
      for (int q0 = 0; q0 < R; q0 += 32) {
        const int rq = std::min(32, R - q0);
        const double* Xq = X + (long long)q0 * n;
        double* Yq = Y + (long long)q0 * n;
        if (rq <= 8)
          k_symm_dmma<8><<<grid, kSyThreads, SymmShape<8>::SMEM, s>>>(ctx->d_A, lda, ctx->d_diag, n, Xq, n, rq, Yq);
        else if (rq <= 16)
          k_symm_dmma<16><<<grid, kSyThreads, SymmShape<16>::SMEM, s>>>(ctx->d_A, lda, ctx->d_diag, n, Xq, n, rq, Yq);
        else if (rq <= 24)
          k_symm_dmma<24><<<grid, kSyThreads, SymmShape<24>::SMEM, s>>>(ctx->d_A, lda, ctx->d_diag, n, Xq, n, rq, Yq);
        else
          k_symm_dmma<32><<<grid, kSyThreads, SymmShape<32>::SMEM, s>>>(ctx->d_A, lda, ctx->d_diag, n, Xq, n, rq, Yq);
        GBEM_LAUNCH_CHECK(ctx);
      }
    } else {
        GBEM_CUDA(ctx, cudaMemsetAsync(Y, 0, sizeof(double) * (size_t)n * R, s));
    int nbt = (n + 63) / 64;
    const dim3 sgrid((unsigned)nbt, (unsigned)std::min(kSymvChunks, nbt));
    for (int q0 = 0; q0 < R; q0 += 8) {
      int rq = std::min(8, R - q0);
      const double* Xq = X + (long long)q0 * n;
      double* Yq = Y + (long long)q0 * n;
      // the narrowest instantiation that holds rq right-hand sides
      if (rq <= 2)
        k_symv_upper<2><<<sgrid, 256, 0, s>>>(ctx->d_A, lda, ctx->d_diag, n, Xq, n, rq, Yq);
      else if (rq <= 4)
        k_symv_upper<4><<<sgrid, 256, 0, s>>>(ctx->d_A, lda, ctx->d_diag, n, Xq, n, rq, Yq);
      else if (rq <= 6)
        k_symv_upper<6><<<sgrid, 256, 0, s>>>(ctx->d_A, lda, ctx->d_diag, n, Xq, n, rq, Yq);
      else
        k_symv_upper<8><<<sgrid, 256, 0, s>>>(ctx->d_A, lda, ctx->d_diag, n, Xq, n, rq, Yq);
      GBEM_LAUNCH_CHECK(ctx);
    }
    }
  return GBEM_OK;
}

// Triangular solves L L^T X = B with the stored factor (gbem_internal_factor),
// residual ||A x - b|| / ||b|| from the preserved upper triangle when d_resid.
int gbem_internal_solve_factored(gbem_ctx* ctx, const double* d_B, int64_t nrhs, double* d_X, double* d_resid,
                                 gbem_solve_stats* stats, bool y_from_border) {
  const int n = (int)ctx->n;
  const long long lda = ctx->lda;
  if (nrhs < 0 || nrhs > (1 << 20)) return ctx->fail(GBEM_EINVAL, "cholesky_solve: nrhs must be in [0, 2^20]");
  if (!ctx->factored) return ctx->fail(GBEM_EINVAL, "no factored matrix in the context");
  if (stats) stats->nrhs = nrhs;
  if (n == 0 || nrhs == 0) return GBEM_OK;
  if (y_from_border && ctx->border != nrhs)
    return ctx->fail(GBEM_EINVAL, "bordered solve: the border does not hold nrhs right-hand sides");
  cudaStream_t s = ctx->stream;
  // forward + backward substitution in one cooperative kernel (a grid barrier
  // per block step instead of four launches per block step)
  const int R = (int)nrhs;
  int rc = ensure_work(ctx, 2 * (size_t)n * (size_t)R);
  if (rc) return rc;
  double* Ysym = ctx->d_work;
  double* scratch = Ysym + (size_t)n * R;
  const double* Linv = ctx->d_linv;
  cudaEventRecord(ctx->ev[1], s);
  static const int blocked_min = getenv("GBEM_SOLVE_BLOCKED_MIN") ? atoi(getenv("GBEM_SOLVE_BLOCKED_MIN")) : 9;
  const int nblk_s = (n + NB - 1) / NB;
  if (y_from_border && R <= 16 && nblk_s <= ctx->num_sms) {
    // bordered factorisation: y is in the border rows; dataflow backward substitution
    if (!ctx->d_flags) {
      GBEM_CUDA(ctx, cudaMalloc(&ctx->d_flags, sizeof(int) * 1024));
      GBEM_CUDA(ctx, cudaMemsetAsync(ctx->d_flags, 0, sizeof(int) * 1024, s));
    }
    if (++ctx->flow_epoch == 0x7fffffff) {
      ctx->flow_epoch = 1;
      GBEM_CUDA(ctx, cudaMemsetAsync(ctx->d_flags, 0, sizeof(int) * 1024, s));
    }
    double* Ys = scratch;
    const long long cnt = (long long)n * R;
    k_border_to_y<<<(unsigned)((cnt + 255) / 256), 256, 0, s>>>(ctx->d_A, lda, n, R, Ys, 0);
    GBEM_LAUNCH_CHECK(ctx);
    const double* cA = ctx->d_A;
    const double* cL = Linv;
    const double* cY = Ys;
    int nn = n, RR = R, ep = ctx->flow_epoch;
    int* fl = ctx->d_flags;
    void* args[] = {(void*)&cA, (void*)&lda, (void*)&cL, (void*)&nn, (void*)&RR, (void*)&cY, (void*)&d_X, (void*)&fl,
                    (void*)&ep};
    void* fn = R <= 2 ? (void*)k_bwd_flow<2> : R <= 4 ? (void*)k_bwd_flow<4> : R <= 6 ? (void*)k_bwd_flow<6>
             : R <= 8 ? (void*)k_bwd_flow<8> : (void*)k_bwd_flow<16>;
    GBEM_CUDA(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFlowSmem));
    GBEM_CUDA(ctx, cudaLaunchCooperativeKernel(fn, dim3(nblk_s), dim3(kFlowThreads), args, kFlowSmem, s));
    GBEM_LAUNCH_CHECK(ctx);
  } else if (y_from_border && R <= kStepRMax && ctx->side_stream && !getenv("GBEM_NO_BWD_LOOKAHEAD")) {
    // bordered, 17..64 right-hand sides (or more blocks than SMs): look-ahead backward substitution
    rc = solve_backward_lookahead(ctx, R, d_X);
    if (rc) return rc;
  } else if (R >= blocked_min || y_from_border) {
    // (bordered: y sits in the border rows; the DMMA-blocked backward sweep takes it for any width)
    rc = solve_blocked(ctx, d_B, R, d_X, y_from_border);
    if (rc) return rc;
  } else {
    const double* cA = ctx->d_A;
    const double* cL = Linv;
    int nn = n;
    static const int dbg = getenv("GBEM_SOLVE_DBG") ? atoi(getenv("GBEM_SOLVE_DBG")) : 0;
    for (int q0 = 0; q0 < R; q0 += kSolveR) {
      int RR = std::min(kSolveR, R - q0);
      const double* Bq = d_B + (size_t)q0 * n;
      double* Xq = d_X + (size_t)q0 * n;
      double* Sq = scratch;  // scratch holds n * R >= n * RR
      int dd = dbg;
      void* args[] = {(void*)&cA, (void*)&lda, (void*)&cL, (void*)&nn, (void*)&RR, (void*)&Bq, (void*)&Xq, (void*)&Sq,
                      (void*)&dd};
      // register blocking over the right-hand sides: the smallest instantiated width >= RR
      void* fn = RR <= 1 ? (void*)k_solve_coop<1> : RR <= 2 ? (void*)k_solve_coop<2> : RR <= 4 ? (void*)k_solve_coop<4>
               : RR <= 6 ? (void*)k_solve_coop<6> : RR <= 8 ? (void*)k_solve_coop<8> : (void*)k_solve_coop<16>;
      GBEM_CUDA(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSolveSmem));
      GBEM_CUDA(ctx, cudaLaunchCooperativeKernel(fn, dim3(ctx->num_sms), dim3(kSolveThreads), args, kSolveSmem, s));
      GBEM_LAUNCH_CHECK(ctx);
    }
  }
  cudaEventRecord(ctx->ev[2], s);
  if (d_resid) {
    rc = apply_sym(ctx, d_X, R, Ysym);
    if (rc) return rc;
    k_resid_norm<<<R, 1024, 0, s>>>(Ysym, d_B, n, d_resid);
    GBEM_LAUNCH_CHECK(ctx);
  }
  cudaEventRecord(ctx->ev[3], s);
  if (stats) {
    GBEM_CUDA(ctx, cudaEventSynchronize(ctx->ev[3]));
    float a = 0, b2 = 0, c = 0;
    (void)a;
    cudaEventElapsedTime(&b2, ctx->ev[1], ctx->ev[2]);
    cudaEventElapsedTime(&c, ctx->ev[2], ctx->ev[3]);
    stats->ms_solve = b2;
    stats->ms_residual = c;
    if (d_resid) {
      std::vector<double> r((size_t)R);
      GBEM_CUDA(ctx, cudaMemcpy(r.data(), d_resid, sizeof(double) * R, cudaMemcpyDeviceToHost));
      double mx = 0;
      for (double v : r) mx = std::max(mx, v);
      stats->max_residual = mx;
    }
  }
  return GBEM_OK;
}

int gbem_internal_apply(gbem_ctx* ctx, const double* d_X, int64_t nrhs, double* d_Y) {
  const int n = (int)ctx->n;
  if (nrhs < 0 || nrhs > (1 << 20)) return ctx->fail(GBEM_EINVAL, "nrhs out of range");
  if (n == 0 || nrhs == 0) return GBEM_OK;
  if (!ctx->factored) {  // the diagonal is still in place: save it for apply_sym
    if (ctx->diag_cap < n) {
      cudaFree(ctx->d_diag);
      GBEM_CUDA(ctx, cudaMalloc(&ctx->d_diag, sizeof(double) * n));
      ctx->diag_cap = n;
    }
    k_save_diag<<<(n + 255) / 256, 256, 0, ctx->stream>>>(ctx->d_A, ctx->lda, n, ctx->d_diag);
    GBEM_LAUNCH_CHECK(ctx);
  }
  return apply_sym(ctx, d_X, (int)nrhs, d_Y);
}

int gbem_internal_solve(gbem_ctx* ctx, const double* d_B, int64_t nrhs, double* d_X, double* d_resid,
                        gbem_solve_stats* stats) {
  if (nrhs < 0 || nrhs > (1 << 20)) return ctx->fail(GBEM_EINVAL, "cholesky_solve: nrhs must be in [0, 2^20]");
  int rc = gbem_internal_factor(ctx, stats);
  if (rc) return rc;
  if (stats) stats->nrhs = nrhs;
  return gbem_internal_solve_factored(ctx, d_B, nrhs, d_X, d_resid, stats);
}

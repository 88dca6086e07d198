// gbem_gemm_sk.cuh — split-K NT DMMA GEMM of the sharded solve (gbem_pcg.cu):
// the row-block product A_r P and the block-Jacobi preconditioner product.
#pragma once
#include <cuda_runtime.h>

#include "gbem_dmma_gemm.cuh"

namespace gbem_sk {

using gbem_gemm::BK;
using gbem_gemm::cp_async16;
using gbem_gemm::cp_async8;
using gbem_gemm::cp_async_commit;
using gbem_gemm::cp_async_wait;
using gbem_gemm::dmma;

// C_z (M x N) = A (M x Kz) * B (N x Kz)^T over the z-th slice of the reduction
// dimension, all column-major: A(i, k) = A[k * lda + i], B(j, k) = B[k * ldb + j],
// C_z(i, j) = C[z * strideC + j * ldc + i].  CTA tile 64 x TN, warps 2 x TN/32
// of 32 x 32 (4 x 4 DMMA m8n8k4 fragments each), BK = 16 slabs in an
// STG-stage cp.async ring.  16-byte copies need even lda / ldb and 16-byte
// aligned bases (vec16), else 8-byte copies.  In the sharded solve M is the
// right-hand-side count (A = the gathered search directions, re-read from L2
// by every CTA) and N the rank's rows (B = the row block, streamed once from
// HBM), so a wider TN halves the L2 re-reads of A per flop.
constexpr int kT = 64;
template <int TN>
struct SkShape {
  static constexpr int THREADS = 2 * TN;           // 2 x TN/32 warps
  static constexpr int LA = kT + 8, LB = TN + 8;   // slab row strides: conflict-free fragment loads
  static constexpr int SLAB = BK * (LA + LB);
  static constexpr int STG = 3;
  static constexpr size_t SMEM = (size_t)STG * SLAB * sizeof(double);
  static constexpr int MINB = TN == 64 ? 4 : 2;
};
constexpr int kThreads = SkShape<64>::THREADS;
constexpr size_t kSmem = SkShape<64>::SMEM;

template <int TN>
static __global__ void __launch_bounds__(SkShape<TN>::THREADS, SkShape<TN>::MINB)
    k_gemm_nt_sk(double* __restrict__ C, long long ldc, long long strideC, const double* __restrict__ A,
                 long long lda, const double* __restrict__ B, long long ldb, int M, int N, long long Ktot,
                 long long kchunk, int vec16) {
  using S = SkShape<TN>;
  extern __shared__ __align__(16) double smem[];
  const int m0 = blockIdx.x * kT, n0 = blockIdx.y * TN;
  const long long kbeg = (long long)blockIdx.z * kchunk;
  const long long kend = min(Ktot, kbeg + kchunk);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int g = lane >> 2, t4 = lane & 3;
  auto load = [&](long long kt, int buf) {
    const long long k0 = kbeg + kt * BK;
    double* as = smem + (size_t)buf * S::SLAB;
    double* bs = as + BK * S::LA;
#pragma unroll
    for (int c = tid; c < BK * kT / 2; c += S::THREADS) {  // A: BK rows (k) x 64
      const int kk = c / (kT / 2), xx = (c % (kT / 2)) * 2;
      const long long gk = k0 + kk;
      const int gm = m0 + xx;
      if (vec16) {
        const bool ok = gk < kend && gm < M;
        cp_async16(as + kk * S::LA + xx, ok ? A + gk * lda + gm : A, ok ? (gm + 1 < M ? 16 : 8) : 0);
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const bool ok = gk < kend && gm + e < M;
          cp_async8(as + kk * S::LA + xx + e, ok ? A + gk * lda + gm + e : A, ok ? 8 : 0);
        }
      }
    }
#pragma unroll
    for (int c = tid; c < BK * TN / 2; c += S::THREADS) {  // B: BK rows (k) x TN
      const int kk = c / (TN / 2), xx = (c % (TN / 2)) * 2;
      const long long gk = k0 + kk;
      const int gn = n0 + xx;
      if (vec16) {
        const bool ok = gk < kend && gn < N;
        cp_async16(bs + kk * S::LB + xx, ok ? B + gk * ldb + gn : B, ok ? (gn + 1 < N ? 16 : 8) : 0);
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const bool ok = gk < kend && gn + e < N;
          cp_async8(bs + kk * S::LB + xx + e, ok ? B + gk * ldb + gn + e : B, ok ? 8 : 0);
        }
      }
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const long long KT = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
#pragma unroll
  for (int s = 0; s < S::STG - 1; ++s) {
    if (s < KT) load(s, s);
    cp_async_commit();
  }
  for (long long kt = 0; kt < KT; ++kt) {
    if (kt + S::STG - 1 < KT) load(kt + S::STG - 1, (int)((kt + S::STG - 1) % S::STG));
    cp_async_commit();
    cp_async_wait<S::STG - 1>();
    __syncthreads();
    const double* as = smem + (size_t)(kt % S::STG) * S::SLAB;
    const double* bs = as + BK * S::LA;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = as[(kk + t4) * S::LA + wm * 32 + i * 8 + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = bs[(kk + t4) * S::LB + wn * 32 + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
  double* Cz = C + (long long)blockIdx.z * strideC;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + wm * 32 + i * 8 + g;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = n0 + wn * 32 + j * 8 + 2 * t4 + e;
        if (col < N) Cz[(long long)col * ldc + row] = acc[i][j][e];
      }
  }
}

// ---------------------------------------------------------------------------
// The same product with bulk-copy (TMA engine) operand staging, as the Cholesky's trailing update
// (gbem_dmma_gemm.cuh, k_syrk_bulk): 64 x 64 tile, 2 x 2 warps, 16-column slabs in a 3-stage
// mbarrier pipeline, every warp issuing a quarter of a slab's 32 copies (512 bytes each), a
// proxy fence before a stage is released.  The slice's last, partial slab is loaded by the
// threads themselves (zero-filled) after the pipeline has drained.  Needs 16-byte aligned
// operands with even leading dimensions and the element after an odd row count readable
// (checked by the launcher, gbem_pcg.cu gemm_nt).
using gbem_gemm::BulkShape;
using gbem_gemm::bulk_g2s;
using gbem_gemm::mbar_arrive;
using gbem_gemm::mbar_expect_tx;
using gbem_gemm::mbar_init;
using gbem_gemm::mbar_wait;

constexpr int kBulkBKS = 16, kBulkNST = 3;
using SkBulk = BulkShape<kBulkBKS, kBulkNST>;

static __global__ void __launch_bounds__(128, 4)
    k_gemm_nt_sk_bulk(double* __restrict__ C, long long ldc, long long strideC, const double* __restrict__ A,
                      long long lda, const double* __restrict__ B, long long ldb, int M, int N, long long Ktot,
                      long long kchunk, int tri = 0) {
  // tri (single-slice products of the block inverse): 1 = A is upper triangular (A(i, k) = 0 for
  // k < i: the tile's reduction starts at its first row), 2 = B is lower triangular (B(j, k) = 0
  // for k > j: it ends with the tile's last row)
  using S = SkBulk;
  constexpr int BKS = kBulkBKS, NST = kBulkNST, T = 64;
  extern __shared__ __align__(16) double smem[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + NST * 2 * S::SLAB);
  unsigned long long* empty = full + NST;
  const int m0 = blockIdx.x * T, n0 = blockIdx.y * T;
  long long kbeg = (long long)blockIdx.z * kchunk;
  long long kend = min(Ktot, kbeg + kchunk);
  if (tri == 1) kbeg = max(kbeg, (long long)m0);
  if (tri == 2) kend = min(kend, (long long)n0 + T);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int g = lane >> 2, t4 = lane & 3;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();
  const long long klen = kend > kbeg ? kend - kbeg : 0;
  const int KT = (int)(klen / BKS);        // full slabs, through the pipeline
  const int ktail = (int)(klen % BKS);     // columns of the last, partial slab
  // this lane's copy: warps 0, 1 the A operand's columns [8 warp, 8 warp + 8), warps 2, 3 B's
  constexpr int kSeg = BKS / 2;
  const int seg = warp * kSeg + (lane % kSeg);
  const bool copier = lane < kSeg;
  const int ck = seg % BKS;
  const bool isA = seg < BKS;
  const int rowsA = min(T, M - m0), rowsB = min(T, N - n0);
  const unsigned bytesA = (unsigned)(((rowsA + 1) & ~1) * 8), bytesB = (unsigned)(((rowsB + 1) & ~1) * 8);
  const unsigned cbytes = isA ? bytesA : bytesB;
  const double* csrc = isA ? A + (kbeg + ck) * lda + m0 : B + (kbeg + ck) * ldb + n0;
  const long long cstep = (isA ? lda : ldb) * BKS;
  const int cdst = (isA ? 0 : S::SLAB) + ck * S::LD;
  const unsigned slab_bytes = (unsigned)BKS * (bytesA + bytesB);
  auto request = [&](int p) {  // every warp
    const int sp = p % NST;
    if (p >= NST) mbar_wait(&empty[sp], ((p / NST) - 1) & 1);
    if (tid == 0) mbar_expect_tx(&full[sp], slab_bytes);
    __syncwarp();
    if (copier) bulk_g2s(smem + sp * 2 * S::SLAB + cdst, csrc + (long long)p * cstep, cbytes, &full[sp]);
  };
#pragma unroll
  for (int p = 0; p < NST - 2; ++p)
    if (p < KT) request(p);
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int aoff = wm * 32 + g, boff = S::SLAB + wn * 32 + g;
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % NST;
    if (kt + NST - 2 < KT) request(kt + NST - 2);
    mbar_wait(&full[s], (kt / NST) & 1);
    const double* as = smem + s * 2 * S::SLAB + aoff;
    const double* bs = smem + s * 2 * S::SLAB + boff;
#pragma unroll
    for (int kk = 0; kk < BKS; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = as[(kk + t4) * S::LD + i * 8];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = bs[(kk + t4) * S::LD + j * 8];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (ktail > 0) {  // block-uniform
    __syncthreads();  // every requested slab has been consumed: no copy is in flight
    const long long k0 = kbeg + (long long)KT * BKS;
    for (int c = tid; c < BKS * T; c += 128) {
      const int kk = c / T, x = c % T;
      const bool kin = kk < ktail;
      smem[kk * S::LD + x] = (kin && m0 + x < M) ? A[(k0 + kk) * lda + m0 + x] : 0.0;
      smem[S::SLAB + kk * S::LD + x] = (kin && n0 + x < N) ? B[(k0 + kk) * ldb + n0 + x] : 0.0;
    }
    __syncthreads();
    const double* as = smem + aoff;
    const double* bs = smem + boff;
    for (int kk = 0; kk < ktail; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = as[(kk + t4) * S::LD + i * 8];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = bs[(kk + t4) * S::LD + j * 8];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  double* Cz = C + (long long)blockIdx.z * strideC;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + wm * 32 + i * 8 + g;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = n0 + wn * 32 + j * 8 + 2 * t4 + e;
        if (col < N) Cz[(long long)col * ldc + row] = acc[i][j][e];
      }
  }
}

}  // namespace gbem_sk

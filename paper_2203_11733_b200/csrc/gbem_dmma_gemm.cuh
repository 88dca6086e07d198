// gbem_dmma_gemm.cuh — FP64 tensor-core (DMMA) GEMM for the Cholesky trailing
// update and the GEMM-form trsm: C (M x N) op= A (M x K) * B (N x K)^T, all
// column-major.  sm_100a has no tcgen05 FP64 kind; the FP64 tensor path is the
// warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), measured at 37.1 TFLOP/s
// (tools/fp64_peaks.cu).
//
// CTA tile 128 x BN, 8 warps as 4 (M) x 2 (N), warp tile 32 x BN/2 =
// 4 x BN/16 DMMA fragments; BK = 16 slabs through a 3-stage cp.async pipeline;
// shared-memory row stride = tile width + 8 doubles makes the 8-byte fragment
// loads conflict-free.  BN = 64 is the trailing-update shape: ~100 registers,
// 80 KB shared memory, two CTAs per SM, so one CTA's epilogue (C read-modify-
// write) and prologue overlap the other's DMMA main loop.  BN = 128 is the
// trsm shape (one CTA owns complete rows, so C may alias A).
//   kSub  : C -= A B^T   (C must not alias A or B)
//   kStore: C  = A B^T
// Tile enumeration (tile_mode): 0 dense grid (blockIdx.x, blockIdx.y);
// 1 every tile touching the lower triangle; 2 tiles with column index < split;
// 3 lower tiles with column index >= split (the look-ahead split of the
// Cholesky: block column k+1 first, then the rest).
#pragma once
#include <cuda_runtime.h>

namespace gbem_gemm {

constexpr int BM = 128, BK = 16, STAGES = 3;
constexpr int GEMM_THREADS = 256;

template <int BN>
struct Shape {
  static constexpr int LDA = BM + 8;  // smem row stride (doubles) of the A slab
  static constexpr int LDB = BN + 8;
  static constexpr int WN = BN / 2;   // warp tile width
  static constexpr int FN = WN / 8;   // DMMA fragments along N per warp
  static constexpr size_t SMEM = (size_t)STAGES * BK * (LDA + LDB) * sizeof(double);
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

enum GemmMode { kSub = 0, kStore = 1 };

// Number of 128 x BN tiles touching the lower triangle in tile row tm (BM = r*BN).
template <int BN>
__host__ __device__ inline long long lower_tiles_before(long long tm) {
  constexpr long long r = BM / BN;  // tile columns per tile row step
  // row tm spans tile columns 0 .. r*tm + r - 1  ->  r*(tm+1) tiles
  return r * tm * (tm + 1) / 2;
}

template <int BN>
__device__ inline void lower_tile(long long t, int split, int mode, int& tm, int& tn) {
  constexpr int r = BM / BN;
  if (mode == 1) {
    // t = r*tm(tm+1)/2 + tn
    int x = (int)((sqrt(8.0 * (double)t / r + 1.0) - 1.0) * 0.5);
    while (lower_tiles_before<BN>(x + 1) <= t) ++x;
    while (lower_tiles_before<BN>(x) > t) --x;
    tm = x;
    tn = (int)(t - lower_tiles_before<BN>(x));
  } else {
    // mode 3: columns >= split (split = r: one block column of 128), rows tm >= 1
    // per row tm: tile columns split .. r*tm + r - 1  ->  r*tm + r - split tiles
    long long lo = 0, hi = 1 << 20;
    while (lo < hi) {  // smallest tm with cum(tm+1) > t
      long long mid = (lo + hi) >> 1;
      long long cum = lower_tiles_before<BN>(mid + 1) - (long long)split * (mid + 1);
      if (cum > t)
        hi = mid;
      else
        lo = mid + 1;
    }
    tm = (int)lo;
    long long before = lower_tiles_before<BN>(lo) - (long long)split * lo;
    tn = split + (int)(t - before);
  }
}

template <int MODE, int BN>
__global__ void __launch_bounds__(GEMM_THREADS, BN == 64 ? 2 : 1)
    k_gemm_nt(double* C, long long ldc, const double* A, long long lda, const double* B, long long ldb, int M,
              int N, int K, int tile_mode, int split) {
  using S = Shape<BN>;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                           // [STAGES][BK][LDA]
  double* Bs = smem + STAGES * BK * S::LDA;    // [STAGES][BK][LDB]
  int tm, tn;
  if (tile_mode == 0) {
    tm = blockIdx.x;
    tn = blockIdx.y;
  } else if (tile_mode == 2) {
    tm = blockIdx.x;
    tn = blockIdx.y;
  } else {
    lower_tile<BN>(blockIdx.x, split, tile_mode, tm, tn);
  }
  const bool lower = tile_mode != 0;
  const int m0 = tm * BM, n0 = tn * BN;
  if (lower && n0 > m0 + BM - 1) return;  // tile entirely above the diagonal
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2;
  const int g = lane >> 2, t4 = lane & 3;

  // kSub starts the accumulators at C (loads issued before the prologue, so
  // their latency overlaps it) and accumulates -A B^T: the epilogue is a
  // plain store and no C read sits after the main loop.
  double acc[4][S::FN][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + wm * 32 + i * 8 + g;
#pragma unroll
    for (int j = 0; j < S::FN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = n0 + wn * S::WN + j * 8 + 2 * t4 + e;
        const bool ok = row < M && col < N && !(lower && col > row);
        acc[i][j][e] = (MODE == kSub && ok) ? C[(long long)col * ldc + row] : 0.0;
      }
  }

  const int KT = (K + BK - 1) / BK;
  auto load_stage = [&](int kt, int st) {
    const int k0 = kt * BK;
    double* as = As + st * BK * S::LDA;
    double* bs = Bs + st * BK * S::LDB;
#pragma unroll
    for (int c = tid; c < BK * BM / 2; c += GEMM_THREADS) {
      int kk = c / (BM / 2), mm = (c % (BM / 2)) * 2;
      int gk = k0 + kk, gm = m0 + mm;
      int bytes = 0;
      const double* src = A;
      if (gk < K && gm < M) {
        bytes = gm + 1 < M ? 16 : 8;
        src = A + (long long)gk * lda + gm;
      }
      cp_async16(as + kk * S::LDA + mm, src, bytes);
    }
#pragma unroll
    for (int c = tid; c < BK * BN / 2; c += GEMM_THREADS) {
      int kk = c / (BN / 2), nn = (c % (BN / 2)) * 2;
      int gk = k0 + kk, gn = n0 + nn;
      int bytes = 0;
      const double* src = B;
      if (gk < K && gn < N) {
        bytes = gn + 1 < N ? 16 : 8;
        src = B + (long long)gk * ldb + gn;
      }
      cp_async16(bs + kk * S::LDB + nn, src, bytes);
    }
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    int nxt = kt + STAGES - 1;
    if (nxt < KT) load_stage(nxt, nxt % STAGES);
    cp_async_commit();
    const double* as = As + (kt % STAGES) * BK * S::LDA;
    const double* bs = Bs + (kt % STAGES) * BK * S::LDB;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[S::FN];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        af[i] = as[(kk + t4) * S::LDA + wm * 32 + i * 8 + g];
        if (MODE == kSub)  // sign flip on the high word: an integer op, not the FP64 pipe
          af[i] = __hiloint2double(__double2hiint(af[i]) ^ (int)0x80000000, __double2loint(af[i]));
      }
#pragma unroll
      for (int j = 0; j < S::FN; ++j) bf[j] = bs[(kk + t4) * S::LDB + wn * S::WN + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < S::FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // epilogue: fragment (i,j) holds rows m0+wm*32+i*8+g, cols n0+wn*WN+j*8+2*t4+{0,1}
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + wm * 32 + i * 8 + g;
#pragma unroll
    for (int j = 0; j < S::FN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = n0 + wn * S::WN + j * 8 + 2 * t4 + e;
        if (row < M && col < N && !(lower && col > row)) C[(long long)col * ldc + row] = acc[i][j][e];
      }
  }
}

__device__ __forceinline__ double neg_hi(double x) {
  return __hiloint2double(__double2hiint(x) ^ (int)0x80000000, __double2loint(x));
}

// ---------------------------------------------------------------------------
// Generic-shape trailing-update kernel (kSub, lower tiles): CTA tile TBM x TBN,
// WMW x WNW warps, warp tile (TBM/WMW) x (TBN/WNW), NSTG-stage cp.async
// pipeline of BK = 16 slabs, accumulators preloaded with C.  Small tiles with
// several CTAs per SM overlap one CTA's prologue/epilogue with the others' DMMA.
#ifndef GBEM_GEN_PAD
#define GBEM_GEN_PAD 8
#endif
template <int TBM, int TBN, int WMW, int WNW, int NSTG>
struct GenShape {
  static constexpr int THREADS = 32 * WMW * WNW;
  static constexpr int LDA = TBM + GBEM_GEN_PAD, LDB = TBN + GBEM_GEN_PAD;
  static constexpr int FM = TBM / WMW / 8, FN = TBN / WNW / 8;
  static constexpr size_t SMEM = (size_t)NSTG * BK * (LDA + LDB) * sizeof(double);
};

template <int TBM, int TBN>
__host__ __device__ inline long long gen_tiles_before(long long tm) {
  constexpr long long r = TBM / TBN;
  return r * tm * (tm + 1) / 2;
}

// Square tiles (TBM == TBN).  band > 0: grid (tile rows, band), tile (x, y)
// with tn = y < band, tm = x (tiles above the diagonal exit) -- the look-ahead
// block column; band == 0: the lower tiles with tile column >= split,
// enumerated triangularly (row tm = split + x holds x + 1 of them).
// band < 0: both in one 1-D grid -- the first nt * (-band) CTAs are the band
// tiles of tile columns [0, -band) (nt = tile rows), dispatched first, then the
// triangle from split = -band; each band CTA bumps *band_done when its tile is
// stored (release), which is what the next diagonal factor waits for.
// Lower-triangle tile t of an X x X tile grid -> (row r, column c), enumerated in column strips
// of kSyrkStrip tile columns, row-major inside a strip: the CTAs in flight at one time then share
// the strip's column operands and a few dozen row operands (~40 MB at K = 1,536 for a strip of 16; 32 measured the same speed), which stay in
// the 126 MB L2.  Plain row-major order walks the whole panel once per tile row; at K >= 640 the
// panel no longer fits the L2 and was re-read from HBM (ncu: 62 GB of DRAM reads for a 0.3 GB
// panel + 2.7 GB of C at m = 26,000, K = 1,536).
#ifndef GBEM_SYRK_STRIP
#define GBEM_SYRK_STRIP 32
#endif
__device__ __forceinline__ void lower_tile_strips(long long t, int X, int& r, int& c) {
#if GBEM_SYRK_STRIP > 0
  constexpr int W = GBEM_SYRK_STRIP;
  int c0 = 0;
  for (;; c0 += W) {
    const int w = min(W, X - c0);
    const long long total = (long long)w * (w + 1) / 2 + (long long)(X - c0 - w) * w;
    if (t < total || c0 + W >= X) {
      const long long tri = (long long)w * (w + 1) / 2;
      if (t < tri) {
        int x = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
        while ((long long)(x + 1) * (x + 2) / 2 <= t) ++x;
        while ((long long)x * (x + 1) / 2 > t) --x;
        r = c0 + x;
        c = c0 + (int)(t - (long long)x * (x + 1) / 2);
      } else {
        t -= tri;
        r = c0 + w + (int)(t / w);
        c = c0 + (int)(t % w);
      }
      return;
    }
    t -= total;
  }
#else
  int x = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((long long)(x + 1) * (x + 2) / 2 <= t) ++x;
  while ((long long)x * (x + 1) / 2 > t) --x;
  r = x;
  c = (int)(t - (long long)x * (x + 1) / 2);
#endif
}

template <int TBM, int TBN, int WMW, int WNW, int NSTG, int MINB>
__global__ void __launch_bounds__(32 * WMW * WNW, MINB)
    k_syrk_gen(double* C, long long ldc, const double* A, long long lda, int M, int K, int split, int band,
               unsigned* band_done = nullptr, long long /* t_off: k_syrk_bulk's signature */ = 0) {
  static_assert(TBM == TBN, "square tiles");
  using S = GenShape<TBM, TBN, WMW, WNW, NSTG>;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + NSTG * BK * S::LDA;
  int tm, tn;
  bool signal = false;
  long long t = blockIdx.x;
  if (band < 0) {
    const int nt = (M + TBM - 1) / TBM;
    if (t < (long long)nt * -band) {
      tm = (int)(t % nt);
      tn = (int)(t / nt);
      signal = true;
      if (tn > tm) {
        if (threadIdx.x == 0) atomicAdd(band_done, 1u);
        return;
      }
    } else {
      t -= (long long)nt * -band;
      split = -band;
      int r, c;
      lower_tile_strips(t, nt - split, r, c);
      tm = split + r;
      tn = split + c;
    }
  } else if (band > 0) {
    tm = blockIdx.x;
    tn = split + blockIdx.y;
    if (tn > tm) return;
  } else {
    int r, c;
    lower_tile_strips(t, (M + TBM - 1) / TBM - split, r, c);
    tm = split + r;
    tn = split + c;
  }
  const int m0 = tm * TBM, n0 = tn * TBN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WMW, wn = warp / WMW;
  const int g = lane >> 2, t4 = lane & 3;
  const int rw0 = m0 + wm * (TBM / WMW), cw0 = n0 + wn * (TBN / WNW);
  // the products are summed first and subtracted from C once at the end (the
  // rounding of C - sum, as in the reference's dot-product form), with the C
  // loads of each fragment row issued together in the epilogue
  double acc[S::FM][S::FN][2];
#pragma unroll
  for (int i = 0; i < S::FM; ++i)
#pragma unroll
    for (int j = 0; j < S::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int KT = (K + BK - 1) / BK;
  auto load_stage = [&](int kt, int st) {
    const int k0 = kt * BK;
    double* as = As + st * BK * S::LDA;
    double* bs = Bs + st * BK * S::LDB;
#pragma unroll
    for (int c = tid; c < BK * TBM / 2; c += S::THREADS) {
      const int kk = c / (TBM / 2), mm = (c % (TBM / 2)) * 2;
      const int gk = k0 + kk, gm = m0 + mm;
      int bytes = 0;
      const double* src = A;
      if (gk < K && gm < M) {
        bytes = gm + 1 < M ? 16 : 8;
        src = A + (long long)gk * lda + gm;
      }
      cp_async16(as + kk * S::LDA + mm, src, bytes);
    }
#pragma unroll
    for (int c = tid; c < BK * TBN / 2; c += S::THREADS) {
      const int kk = c / (TBN / 2), nn = (c % (TBN / 2)) * 2;
      const int gk = k0 + kk, gn = n0 + nn;
      int bytes = 0;
      const double* src = A;
      if (gk < K && gn < M) {
        bytes = gn + 1 < M ? 16 : 8;
        src = A + (long long)gk * lda + gn;
      }
      cp_async16(bs + kk * S::LDB + nn, src, bytes);
    }
  };
#pragma unroll
  for (int st = 0; st < NSTG - 1; ++st) {
    if (st < KT) load_stage(st, st);
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
#if !defined(GBEM_EXP_NOSYNC)
    cp_async_wait<NSTG - 2>();
    __syncthreads();
#endif
    const int nxt = kt + NSTG - 1;
#if !defined(GBEM_EXP_NOLOAD)
    if (nxt < KT) load_stage(nxt, nxt % NSTG);
    cp_async_commit();
#endif
    const double* as = As + (kt % NSTG) * BK * S::LDA + (wm * (TBM / WMW)) + g;
    const double* bs = Bs + (kt % NSTG) * BK * S::LDB + (wn * (TBN / WNW)) + g;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[S::FM], bf[S::FN];
#pragma unroll
      for (int i = 0; i < S::FM; ++i) af[i] = as[(kk + t4) * S::LDA + i * 8];
#pragma unroll
      for (int j = 0; j < S::FN; ++j) bf[j] = bs[(kk + t4) * S::LDB + j * 8];
#pragma unroll
      for (int i = 0; i < S::FM; ++i)
#pragma unroll
        for (int j = 0; j < S::FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < S::FM; ++i) {
    const int row = rw0 + i * 8 + g;
    double cur[S::FN][2];
#pragma unroll
    for (int j = 0; j < S::FN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = cw0 + j * 8 + 2 * t4 + e;
        cur[j][e] = (row < M && col <= row) ? C[(long long)col * ldc + row] : 0.0;
      }
#pragma unroll
    for (int j = 0; j < S::FN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = cw0 + j * 8 + 2 * t4 + e;
        if (row < M && col <= row) C[(long long)col * ldc + row] = cur[j][e] - acc[i][j][e];
      }
  }
  if (signal) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(band_done, 1u);
  }
}

// ---------------------------------------------------------------------------
// Trailing update with bulk-copy (TMA engine) operand staging.  Same tiles, warp layout, DMMA
// order and rounding as k_syrk_gen<64, 64, 2, 2, ., .>, but the operand slabs are not fetched by
// the DMMA warps' own cp.async (LDGSTS) instructions: measured on a B200 (tools/sync_ab.sh) the
// update runs at 34.3 TFLOP/s with those loads, 36.4 with them removed and 34.2 with only the
// block barrier removed -- the LDGSTS stream (8 per thread per 16-column slab, plus addresses and
// predicates) costs the DMMA pipe 6%, the barrier nothing.  Here one warp per slab (rotating)
// issues a single predicated cp.async.bulk: lanes 0 .. BKS-1 each copy one 64-double column
// segment of the row operand, lanes BKS .. 2 BKS - 1 one of the column operand (512 bytes each,
// SASS UBLKCP) into a padded slab (row stride 68 doubles: conflict-free fragment loads); the
// copies signal a per-stage "full" mbarrier (expect_tx), the four warps release a stage through
// an "empty" mbarrier, and a slab is requested two slabs ahead of its use so a lagging warp does
// not stall the producer.  Requirements (checked by the host launcher, which falls back to
// k_syrk_gen): K % BKS == 0, lda even, 16-byte aligned operands, and the element after an odd row
// count readable (the copies are rounded up to 16 bytes; the extra value only reaches accumulator
// rows >= M, which are never stored).
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  do {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int BKS, int NST>
struct BulkShape {
  static constexpr int T = 64, THREADS = 128, LD = T + 4;
  static constexpr int SLAB = BKS * LD;  // doubles per operand slab
  static constexpr size_t SMEM = (size_t)NST * 2 * SLAB * sizeof(double) + 2 * NST * sizeof(unsigned long long);
  static_assert(2 * BKS <= 32 && BKS % 4 == 0, "one copy per lane");
  static_assert(NST >= 3, "slabs are requested NST - 2 ahead");
};

// TRI_STORE: C = A A^T (lower tiles, stored, C not read) for an upper-triangular A -- tile (tm, tn)
// starts its reduction at column 64 tm, the first one where rows >= 64 tm of A are non-zero (the
// block-Jacobi inverses of the sharded solve: inv(M) = N N^T with N = -inv(L)^T).
template <int BKS, int NST, int MINB, bool SPLIT = false, bool TRI_STORE = false>
__global__ void __launch_bounds__(128, MINB)
    k_syrk_bulk(double* C, long long ldc, const double* A, long long lda, int M, int K, int split, int band,
                unsigned* band_done = nullptr, long long t_off = 0) {
  using S = BulkShape<BKS, NST>;
  constexpr int T = S::T;
  extern __shared__ __align__(16) double smem[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + NST * 2 * S::SLAB);
  unsigned long long* empty = full + NST;
  int tm, tn;
  bool signal = false;
  long long t = blockIdx.x + t_off;  // t_off: this launch covers tiles [t_off, t_off + gridDim.x) of the enumeration
  if (band < 0) {
    const int nt = (M + T - 1) / T;
    if (t < (long long)nt * -band) {
      tm = (int)(t % nt);
      tn = (int)(t / nt);
      signal = true;
      if (tn > tm) {
        if (threadIdx.x == 0) atomicAdd(band_done, 1u);
        return;
      }
    } else {
      t -= (long long)nt * -band;
      split = -band;
      int r, c;
      lower_tile_strips(t, nt - split, r, c);
      tm = split + r;
      tn = split + c;
    }
  } else if (band > 0) {
    tm = blockIdx.x;
    tn = split + blockIdx.y;
    if (tn > tm) return;
  } else {
    int r, c;
    lower_tile_strips(t, (M + T - 1) / T - split, r, c);
    tm = split + r;
    tn = split + c;
  }
  const int m0 = tm * T, n0 = tn * T;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int g = lane >> 2, t4 = lane & 3;
  const int rw0 = m0 + wm * 32, cw0 = n0 + wn * 32;
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
  // this lane's copy.  One warp per slab (SPLIT = false): lanes [0, BKS) the row operand's column
  // k0 + lane, [BKS, 2 BKS) the column operand's.  SPLIT: every warp copies a quarter of each slab
  // (segment warp * BKS / 2 + lane, lanes [0, BKS / 2)) and arrives on the full barrier itself.
  constexpr int kSeg = SPLIT ? BKS / 2 : 2 * BKS;       // segments per producing warp
  const int seg = SPLIT ? warp * kSeg + (lane % kSeg) : lane % kSeg;
  const bool copier = lane < kSeg;
  const int ck = seg % BKS;
  const int crow = seg < BKS ? m0 : n0;
  const int crows = min(T, M - crow);  // >= 1: both tile origins are below M
  const unsigned cbytes = (unsigned)(((crows + 1) & ~1) * 8);
  const int kt0 = TRI_STORE ? m0 / BKS : 0;  // slabs skipped (zero rows of a triangular operand)
  const double* csrc = A + ((long long)kt0 * BKS + ck) * lda + crow;
  const int cdst = (seg < BKS ? 0 : S::SLAB) + ck * S::LD;
  // bytes of one whole slab (both operands); one thread (warp 0's lane 0 when SPLIT, else the
  // producing warp's) posts them on the stage's full barrier, every copy subtracts its own
  const unsigned slab_bytes =
      (unsigned)BKS * 8u * (unsigned)(((min(T, M - m0) + 1) & ~1) + ((min(T, M - n0) + 1) & ~1));
  const int KT = K / BKS - kt0;
  auto request = [&](int p) {  // whole warp
    const int sp = p % NST;
    if (p >= NST) mbar_wait(&empty[sp], ((p / NST) - 1) & 1);
    if (lane == 0 && (!SPLIT || warp == 0)) mbar_expect_tx(&full[sp], slab_bytes);
    __syncwarp();
    if (copier) bulk_g2s(smem + sp * 2 * S::SLAB + cdst, csrc + (long long)p * BKS * lda, cbytes, &full[sp]);
  };
  if (SPLIT || warp == 0) {
#pragma unroll
    for (int p = 0; p < NST - 2; ++p)
      if (p < KT) request(p);
  }
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int aoff = wm * 32 + g, boff = S::SLAB + wn * 32 + g;
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % NST;
    if ((SPLIT || warp == (kt & 3)) && kt + NST - 2 < KT) request(kt + NST - 2);
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
#ifndef GBEM_BULK_NOFENCE
    // the stage is re-filled through the async proxy: order this warp's (generic-proxy) fragment
    // loads before that write
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
#endif
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = rw0 + i * 8 + g;
    double cur[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = cw0 + j * 8 + 2 * t4 + e;
        cur[j][e] = (!TRI_STORE && row < M && col <= row) ? C[(long long)col * ldc + row] : 0.0;
      }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = cw0 + j * 8 + 2 * t4 + e;
        if (row < M && col <= row) C[(long long)col * ldc + row] = TRI_STORE ? acc[i][j][e] : cur[j][e] - acc[i][j][e];
      }
  }
  if (signal) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(band_done, 1u);
  }
}

// ---------------------------------------------------------------------------
// Panel trsm of the Cholesky as a GEMM on 32-row strips: C = A B^T with A the
// M x K strip (column-major, lda), B the N x K inverse of the diagonal factor
// (column-major, ldb), N, K <= 128; C may alias A (a CTA reads its whole strip
// before it writes).  One CTA of 4 warps per 32 rows, warp w owns columns
// [32 w, 32 w + 32).  The footprint (<= 128 registers x 128 threads, 34 KB of
// shared memory in BK = 8 slabs) is at most one trailing-update CTA's, so on a
// high-priority stream a strip takes the first update slot that frees up
// instead of waiting for an SM to drain.
constexpr int kTrsmRows = 32, kTrsmThreads = 128, kTrsmStages = 3, kTrsmBK = 8;
constexpr int kTrsmLA = kTrsmRows + 8, kTrsmLB = 128 + 8;
constexpr size_t kTrsmSmem = (size_t)kTrsmStages * kTrsmBK * (kTrsmLA + kTrsmLB) * sizeof(double);

static __global__ void __launch_bounds__(kTrsmThreads, 4)
    k_trsm_rows(double* C, long long ldc, const double* A, long long lda, const double* __restrict__ B,
                long long ldb, int M, int N, int K) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                                      // [stages][BK][kTrsmLA]
  double* Bs = smem + kTrsmStages * kTrsmBK * kTrsmLA;    // [stages][BK][kTrsmLB]
  const int m0 = blockIdx.x * kTrsmRows;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int KT = (K + kTrsmBK - 1) / kTrsmBK;
  auto load_stage = [&](int kt, int st) {
    const int k0 = kt * kTrsmBK;
    double* as = As + st * kTrsmBK * kTrsmLA;
    double* bs = Bs + st * kTrsmBK * kTrsmLB;
    {  // A: 8 x 32 doubles = 128 16-byte chunks, 1 per thread
      const int kk = tid / (kTrsmRows / 2), mm = (tid % (kTrsmRows / 2)) * 2;
      const int gk = k0 + kk, gm = m0 + mm;
      int bytes = 0;
      const double* src = A;
      if (gk < K && gm < M) {
        bytes = gm + 1 < M ? 16 : 8;
        src = A + (long long)gk * lda + gm;
      }
      cp_async16(as + kk * kTrsmLA + mm, src, bytes);
    }
#pragma unroll
    for (int c = tid; c < kTrsmBK * 128 / 2; c += kTrsmThreads) {  // B: 8 x 128, 4 per thread
      const int kk = c / 64, nn = (c % 64) * 2;
      const int gk = k0 + kk;
      int bytes = 0;
      const double* src = B;
      if (gk < K && nn < N) {
        bytes = nn + 1 < N ? 16 : 8;
        src = B + (long long)gk * ldb + nn;
      }
      cp_async16(bs + kk * kTrsmLB + nn, src, bytes);
    }
  };
#pragma unroll
  for (int st = 0; st < kTrsmStages - 1; ++st) {
    if (st < KT) load_stage(st, st);
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<kTrsmStages - 2>();
    __syncthreads();
    const int nxt = kt + kTrsmStages - 1;
    if (nxt < KT) load_stage(nxt, nxt % kTrsmStages);
    cp_async_commit();
    const double* as = As + (kt % kTrsmStages) * kTrsmBK * kTrsmLA + g;
    const double* bs = Bs + (kt % kTrsmStages) * kTrsmBK * kTrsmLB + warp * 32 + g;
#pragma unroll
    for (int kk = 0; kk < kTrsmBK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = as[(kk + t4) * kTrsmLA + i * 8];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = bs[(kk + t4) * kTrsmLB + j * 8];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // every warp's reads of the strip precede any write (C may alias A)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + i * 8 + g;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = warp * 32 + j * 8 + 2 * t4 + e;
        if (row < M && col < N) C[(long long)col * ldc + row] = acc[i][j][e];
      }
  }
}

// ---------------------------------------------------------------------------
// General dense DMMA GEMM on 64 x 64 tiles (2 x 2 warps of 32 x 32, 4 CTAs/SM,
// double-buffered BK = 16 slabs), for the blocked multi-right-hand-side solves:
//   C (M x N) op= A (M x K) * op(B),  A column-major (lda),
//   BT = 0: op(B) = B^T with B N x K column-major (ldb)   ("NT")
//   BT = 1: op(B) = B   with B K x N column-major (ldb)   ("NN")
//   MODE kSub: C -= A op(B) (products summed, subtracted once); kStore: C = A op(B).
// 16-byte cp.async when the leading dimensions and base pointers allow it
// (vec16), else element-wise 8-byte copies.
constexpr int kGT = 64;             // tile edge
constexpr int kGThreads = 128;
constexpr int kGLA = kGT + 8;       // A slab [BK][64 + 8]
constexpr int kGLBt = kGT + 8;      // NT: B slab [BK][64 + 8]
constexpr int kGLBn = BK + 4;       // NN: B slab [64][BK + 4] (k contiguous)
constexpr size_t kGSmem = (size_t)2 * (BK * kGLA + (kGT * kGLBn > BK * kGLBt ? kGT * kGLBn : BK * kGLBt)) * sizeof(double);

template <int MODE, int BT>
__global__ void __launch_bounds__(kGThreads, 4)
    k_gemm_g(double* __restrict__ C, long long ldc, const double* __restrict__ A, long long lda,
             const double* __restrict__ B, long long ldb, int M, int N, int K, int vec16) {
  constexpr int SA = BK * kGLA;
  constexpr int SB = (kGT * kGLBn > BK * kGLBt ? kGT * kGLBn : BK * kGLBt);
  extern __shared__ __align__(16) double smem[];
  double* As = smem;           // [2][SA]
  double* Bs = smem + 2 * SA;  // [2][SB]
  const int m0 = blockIdx.x * kGT, n0 = blockIdx.y * kGT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int g = lane >> 2, t4 = lane & 3;
  auto load = [&](int kt, int buf) {
    const int k0 = kt * BK;
    double* as = As + buf * SA;
    double* bs = Bs + buf * SB;
    for (int c = tid; c < BK * kGT / 2; c += kGThreads) {  // A: BK rows (k) x 64 (m)
      const int kk = c / (kGT / 2), mm = (c % (kGT / 2)) * 2;
      const int gk = k0 + kk, gm = m0 + mm;
      if (vec16) {
        const bool ok = gk < K && gm < M;
        cp_async16(as + kk * kGLA + mm, ok ? A + (long long)gk * lda + gm : A, ok ? (gm + 1 < M ? 16 : 8) : 0);
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const bool ok = gk < K && gm + e < M;
          cp_async8(as + kk * kGLA + mm + e, ok ? A + (long long)gk * lda + gm + e : A, ok ? 8 : 0);
        }
      }
    }
    if (BT == 0) {
      for (int c = tid; c < BK * kGT / 2; c += kGThreads) {  // B (N x K): BK rows (k) x 64 (n)
        const int kk = c / (kGT / 2), nn = (c % (kGT / 2)) * 2;
        const int gk = k0 + kk, gn = n0 + nn;
        if (vec16) {
          const bool ok = gk < K && gn < N;
          cp_async16(bs + kk * kGLBt + nn, ok ? B + (long long)gk * ldb + gn : B, ok ? (gn + 1 < N ? 16 : 8) : 0);
        } else {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const bool ok = gk < K && gn + e < N;
            cp_async8(bs + kk * kGLBt + nn + e, ok ? B + (long long)gk * ldb + gn + e : B, ok ? 8 : 0);
          }
        }
      }
    } else {
      for (int c = tid; c < kGT * BK / 2; c += kGThreads) {  // B (K x N): 64 rows (n) x BK (k)
        const int nn = c / (BK / 2), kk = (c % (BK / 2)) * 2;
        const int gk = k0 + kk, gn = n0 + nn;
        if (vec16) {
          const bool ok = gn < N && gk < K;
          cp_async16(bs + nn * kGLBn + kk, ok ? B + (long long)gn * ldb + gk : B, ok ? (gk + 1 < K ? 16 : 8) : 0);
        } else {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const bool ok = gn < N && gk + e < K;
            cp_async8(bs + nn * kGLBn + kk + e, ok ? B + (long long)gn * ldb + gk + e : B, ok ? 8 : 0);
          }
        }
      }
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int KT = (K + BK - 1) / BK;
  if (KT > 0) load(0, 0);
  cp_async_commit();
  for (int kt = 0; kt < KT; ++kt) {
    if (kt + 1 < KT) load(kt + 1, (kt + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* as = As + (kt & 1) * SA + wm * 32 + g;
    const double* bs = Bs + (kt & 1) * SB;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = as[(kk + t4) * kGLA + i * 8];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        bf[j] = BT == 0 ? bs[(kk + t4) * kGLBt + wn * 32 + j * 8 + g] : bs[(wn * 32 + j * 8 + g) * kGLBn + kk + t4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + wm * 32 + i * 8 + g;
    if (row >= M) continue;
    double cur[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = n0 + wn * 32 + j * 8 + 2 * t4 + e;
        cur[j][e] = (MODE == kSub && col < N) ? C[(long long)col * ldc + row] : 0.0;
      }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = n0 + wn * 32 + j * 8 + 2 * t4 + e;
        if (col < N) C[(long long)col * ldc + row] = MODE == kSub ? cur[j][e] - acc[i][j][e] : acc[i][j][e];
      }
  }
}

}  // namespace gbem_gemm

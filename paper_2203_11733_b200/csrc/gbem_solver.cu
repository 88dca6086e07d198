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
//   k_gemm_nt<STORE,128>: L21 = A21 * inv(L11)^T (trsm as a DMMA GEMM, in place);
//   k_gemm_nt<SUB,64>   : A22 -= L21 * L21^T on lower 128x64 tiles (the O(n^3) part).
#include <algorithm>
#include <cmath>
#include <vector>

#include "gbem_ctx.cuh"
#include "gbem_dmma_gemm.cuh"

namespace {

using namespace gbem_gemm;
constexpr int NB = 128;       // Cholesky block size
// Factor the kb x kb diagonal block at A (lda) in shared memory and, in the
// same column sweep, form X = inv(L11) (forward substitution on the identity
// interleaved with the factorisation), one __syncthreads per column:
//   phase j: with s_j = sqrt(a_jj) (column j still unscaled),
//     a(r,c) -= a(r,j) a(c,j) / a_jj           j < c <= r   (Cholesky trailing update)
//     S(r,c) -= a(r,j) S(j,c) / a_jj            c < j < r    (X rows, S = X * diag(L))
//     S(r,j)  = -a(r,j) / a_jj                  j < r
//   and column j-1 / row j-1 are finalised (scaled by 1/s_{j-1}) in the same
//   phase, since phase j never touches them.  X's strict lower part is kept
//   transposed in the strict upper half of the smem tile, its diagonal in xd.
// L11 goes back to A (lower), X to Linv (column-major, ld = NB) for the
// GEMM-form trsm and the triangular solves.  info[0] receives the first failing
// global row (atomicMin); a failed pivot continues as 1 so the launch sequence
// stays fixed (the caller reports "matrix not positive definite").
__global__ void __launch_bounds__(512)
    k_potrf_diag(double* A, long long lda, int kb, int row0, double* Linv, int* info) {
  extern __shared__ __align__(16) double sm[];
  constexpr int LD = NB + 1;
  double* a = sm;               // [NB][LD] column-major: a[c*LD + r]
  double* isq = sm + NB * LD;   // 1/s_j per column
  double* sq = isq + NB;        // s_j
  const int tid = threadIdx.x;
  const int tx = tid & 31, ty = tid >> 5, nty = blockDim.x >> 5;
  for (int idx = tid; idx < kb * kb; idx += blockDim.x) {
    int c = idx / kb, r = idx % kb;
    a[c * LD + r] = r >= c ? A[(long long)c * lda + r] : 0.0;
  }
  __syncthreads();
  bool bad = false;
  for (int j = 0; j < kb; ++j) {
    double d = a[j * LD + j];
    if (!(d > 0.0)) {
      if (tid == 0 && !bad) atomicMin(info, row0 + j);
      bad = true;
      d = 1.0;
    }
    const double sj = sqrt(d), inv_s = 1.0 / sj, inv_d = inv_s * inv_s;
    if (tid == 0) {
      isq[j] = inv_s;
      sq[j] = sj;
    }
    // finalise column j-1 of L and row j-1 of X
    if (j > 0) {
      const int p = j - 1;
      const double ip = isq[p];
      for (int r = p + 1 + tid; r < kb; r += blockDim.x) a[p * LD + r] *= ip;  // L(r,p)
      for (int c = tid; c < p; c += blockDim.x) a[p * LD + c] *= ip;          // X(p,c) stored at (c,p)
    }
    for (int r = j + 1 + ty; r < kb; r += nty) {
      const double arj = a[j * LD + r] * inv_d;
      for (int c = tx; c <= r; c += 32) {
        if (c > j)
          a[c * LD + r] -= arj * a[j * LD + c];       // trailing Cholesky update
        else if (c < j)
          a[r * LD + c] -= arj * a[j * LD + c];       // S(r,c) -= L(r,j) X(j,c)   (stored at (c,r))
        else
          a[r * LD + j] = -arj;                        // S(r,j) = -L(r,j) / L(j,j)
      }
    }
    __syncthreads();
  }
  if (kb > 0) {
    const int p = kb - 1;
    const double ip = isq[p];
    for (int c = tid; c < p; c += blockDim.x) a[p * LD + c] *= ip;
  }
  __syncthreads();
  for (int idx = tid; idx < kb * kb; idx += blockDim.x) {
    int c = idx / kb, r = idx % kb;
    if (r > c) A[(long long)c * lda + r] = a[c * LD + r];
    else if (r == c) A[(long long)c * lda + r] = sq[r];
  }
  for (int idx = tid; idx < NB * NB; idx += blockDim.x) {
    int c = idx / NB, r = idx % NB;
    double v = 0.0;
    if (r < kb && c < kb) {
      if (r > c) v = a[r * LD + c];
      else if (r == c) v = isq[r];
    }
    Linv[c * NB + r] = v;
  }
}

// Forward step: Y_k = inv(L_kk) B_k (B_k overwritten), rows [k0, k0+kb), all rhs.
__global__ void k_trsv_diag(const double* Linv, int kb, double* B, long long ldb, int k0, int nrhs,
                            int transpose) {
  __shared__ double y[NB];
  for (int r = blockIdx.x; r < nrhs; r += gridDim.x) {
    double* b = B + (long long)r * ldb + k0;
    for (int i = threadIdx.x; i < kb; i += blockDim.x) y[i] = b[i];
    __syncthreads();
    for (int i = threadIdx.x; i < kb; i += blockDim.x) {
      double s = 0.0;
      if (!transpose) {
        for (int k = 0; k <= i; ++k) s += Linv[k * NB + i] * y[k];  // (Linv)(i,k)
      } else {
        for (int k = i; k < kb; ++k) s += Linv[i * NB + k] * y[k];  // (Linv^T)(i,k) = Linv(k,i)
      }
      b[i] = s;
    }
    __syncthreads();
  }
}

// Forward update: B[r] -= sum_{c in block} L(r, c) Y[c] for rows r >= k0+kb.
// Thread per row (coalesced over r for each c), nrhs accumulators in registers.
template <int MAXR>
__global__ void k_fwd_update(const double* A, long long lda, int k0, int kb, int n, double* B,
                             long long ldb, int nrhs) {
  __shared__ double ys[NB * MAXR];
  for (int idx = threadIdx.x; idx < kb * nrhs; idx += blockDim.x) {
    int c = idx % kb, rr = idx / kb;
    ys[c * MAXR + rr] = B[(long long)rr * ldb + k0 + c];
  }
  __syncthreads();
  int r = k0 + kb + blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double acc[MAXR];
#pragma unroll
  for (int q = 0; q < MAXR; ++q) acc[q] = 0.0;
  for (int c = 0; c < kb; ++c) {
    double l = A[(long long)(k0 + c) * lda + r];
#pragma unroll
    for (int q = 0; q < MAXR; ++q) acc[q] = fma(l, ys[c * MAXR + q], acc[q]);
  }
#pragma unroll
  for (int q = 0; q < MAXR; ++q)
    if (q < nrhs) B[(long long)q * ldb + r] -= acc[q];
}

// Backward update: Y[r] -= sum_{c in block k} L(c, r) X[c] for rows r < k0.
// L(c, r) (row c in block k, col r) sits at A[r*lda + c]: a warp reads the
// kb-long contiguous column segment of row r.
template <int MAXR>
__global__ void k_bwd_update(const double* A, long long lda, int k0, int kb, double* B, long long ldb,
                             int nrhs) {
  __shared__ double xs[NB * MAXR];
  for (int idx = threadIdx.x; idx < kb * nrhs; idx += blockDim.x) {
    int c = idx % kb, rr = idx / kb;
    xs[c * MAXR + rr] = B[(long long)rr * ldb + k0 + c];
  }
  __syncthreads();
  int lane = threadIdx.x & 31;
  int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= k0) return;
  double acc[MAXR];
#pragma unroll
  for (int q = 0; q < MAXR; ++q) acc[q] = 0.0;
  for (int c = lane; c < kb; c += 32) {
    double l = A[(long long)r * lda + k0 + c];
#pragma unroll
    for (int q = 0; q < MAXR; ++q) acc[q] = fma(l, xs[c * MAXR + q], acc[q]);
  }
#pragma unroll
  for (int q = 0; q < MAXR; ++q) {
    double v = acc[q];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0 && q < nrhs) B[(long long)q * ldb + r] -= v;
  }
}

__global__ void k_save_diag(const double* A, long long lda, int n, double* d) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[i] = A[(long long)i * lda + i];
}

// y = A x with A given by its strict upper triangle (col-major, A[c*lda + r],
// r < c) and the saved diagonal; 64 x 64 tiles (I <= J), atomics into y.
template <int MAXR>
__global__ void k_symv_upper(const double* A, long long lda, const double* diag, int n,
                             const double* X, long long ldx, int nrhs, double* Y) {
  constexpr int T = 64;
  long long t = blockIdx.x;
  int nbt = (n + T - 1) / T;
  // upper tile (bi <= bj) from linear index, row-major over bi
  int bi = 0;
  long long off = 0;
  while (off + (nbt - bi) <= t) {
    off += nbt - bi;
    ++bi;
  }
  int bj = bi + (int)(t - off);
  __shared__ double xi[T * MAXR], xj[T * MAXR];
  for (int idx = threadIdx.x; idx < T * nrhs; idx += blockDim.x) {
    int r = idx % T, q = idx / T;
    int gi = bi * T + r, gj = bj * T + r;
    xi[r * MAXR + q] = gi < n ? X[(long long)q * ldx + gi] : 0.0;
    xj[r * MAXR + q] = gj < n ? X[(long long)q * ldx + gj] : 0.0;
  }
  __syncthreads();
  // thread per column c of the tile (T threads): y_j[c] += sum_r A(r,c) x_i[r];
  // and per row r: y_i[r] += sum_c A(r,c) x_j[c] (second pass)
  int tid = threadIdx.x;
  if (tid < T) {
    int c = bj * T + tid;
    if (c < n) {
      double acc[MAXR];
#pragma unroll
      for (int q = 0; q < MAXR; ++q) acc[q] = 0.0;
      for (int rr = 0; rr < T; ++rr) {
        int r = bi * T + rr;
        if (r >= n || r >= c) break;
        double a = A[(long long)c * lda + r];
#pragma unroll
        for (int q = 0; q < MAXR; ++q) acc[q] = fma(a, xi[rr * MAXR + q], acc[q]);
      }
      if (bi == bj) {
#pragma unroll
        for (int q = 0; q < MAXR; ++q) acc[q] = fma(diag[c], xj[tid * MAXR + q], acc[q]);
      }
#pragma unroll
      for (int q = 0; q < MAXR; ++q)
        if (q < nrhs) atomicAdd(&Y[(long long)q * n + c], acc[q]);
    }
  } else if (tid < 2 * T) {
    int rr = tid - T;
    int r = bi * T + rr;
    if (r < n) {
      double acc[MAXR];
#pragma unroll
      for (int q = 0; q < MAXR; ++q) acc[q] = 0.0;
      for (int cc = 0; cc < T; ++cc) {
        int c = bj * T + cc;
        if (c >= n) break;
        if (c <= r) continue;
        double a = A[(long long)c * lda + r];
#pragma unroll
        for (int q = 0; q < MAXR; ++q) acc[q] = fma(a, xj[cc * MAXR + q], acc[q]);
      }
#pragma unroll
      for (int q = 0; q < MAXR; ++q)
        if (q < nrhs) atomicAdd(&Y[(long long)q * n + r], acc[q]);
    }
  }
}

// resid[q] = ||Y[:,q] - B[:,q]|| / ||B[:,q]|| (one CTA per rhs)
__global__ void k_resid_norm(const double* Y, const double* B, int n, double* resid) {
  int q = blockIdx.x;
  double rn = 0.0, bn = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double d = Y[(long long)q * n + i] - B[(long long)q * n + i];
    double b = B[(long long)q * n + i];
    rn += d * d;
    bn += b * b;
  }
  __shared__ double s1[256], s2[256];
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

__global__ void k_copy(const double* src, double* dst, long long count) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < count) dst[i] = src[i];
}

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

// Blocked Cholesky of ctx->d_A (n x n) + solves for nrhs columns of d_B (ld n)
// into d_X; d_resid[nrhs] optional.
int gbem_internal_solve(gbem_ctx* ctx, const double* d_B, int64_t nrhs, double* d_X, double* d_resid,
                        gbem_solve_stats* stats) {
  const int n = (int)ctx->n;
  const long long lda = ctx->lda;
  if (stats) {
    *stats = gbem_solve_stats{};
    stats->n = n;
    stats->nrhs = nrhs;
    stats->bad_pivot = -1;
  }
  if (nrhs < 0 || nrhs > 64) return ctx->fail(GBEM_EINVAL, "cholesky_solve: nrhs must be in [0, 64]");
  if (n == 0) return GBEM_OK;
  if (ctx->factored) return ctx->fail(GBEM_EINVAL, "matrix already factored; re-assemble or re-upload");
  const int nblk = (n + NB - 1) / NB;
  // workspace: inverses of the diagonal blocks (nblk * NB * NB) + symv result (n * nrhs)
  size_t need = (size_t)nblk * NB * NB + (size_t)n * (size_t)std::max<int64_t>(nrhs, 1);
  int rc = ensure_work(ctx, need);
  if (rc) return rc;
  double* Linv = ctx->d_work;
  double* Ysym = ctx->d_work + (size_t)nblk * NB * NB;
  if (ctx->diag_cap < n) {
    if (ctx->d_diag) cudaFree(ctx->d_diag);
    GBEM_CUDA(ctx, cudaMalloc(&ctx->d_diag, sizeof(double) * n));
    ctx->diag_cap = n;
  }
  if (!ctx->d_info) {
    GBEM_CUDA(ctx, cudaMalloc(&ctx->d_info, sizeof(int)));
    GBEM_CUDA(ctx, cudaMallocHost(&ctx->h_info, sizeof(int)));
  }
  static bool attr_done = false;
  if (!attr_done) {
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_gemm_nt<kSub, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)Shape<64>::SMEM));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_gemm_nt<kStore, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)Shape<128>::SMEM));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_potrf_diag, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)((NB * (NB + 1) + 2 * NB) * sizeof(double))));
    attr_done = true;
  }
  cudaStream_t s = ctx->stream;
  int big = 0x7fffffff;
  GBEM_CUDA(ctx, cudaMemcpyAsync(ctx->d_info, &big, sizeof(int), cudaMemcpyHostToDevice, s));
  k_save_diag<<<(n + 255) / 256, 256, 0, s>>>(ctx->d_A, lda, n, ctx->d_diag);
  GBEM_LAUNCH_CHECK(ctx);
  cudaEventRecord(ctx->ev[0], s);
  const size_t potrf_smem = (size_t)(NB * (NB + 1) + 2 * NB) * sizeof(double);
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
  cudaStream_t s1 = ctx->side_stream;
  GBEM_CUDA(ctx, cudaEventRecord(ctx->ev_col, s));
  for (int b = 0; b < nblk; ++b) {
    int k0 = b * NB, kb = std::min(NB, n - k0);
    int m = n - k0 - kb;
    double* Akk = ctx->d_A + (long long)k0 * lda + k0;
    double* A21 = Akk + kb;  // rows k0+kb.., cols k0..
    GBEM_CUDA(ctx, cudaStreamWaitEvent(s1, ctx->ev_col, 0));
    k_potrf_diag<<<1, 512, potrf_smem, s1>>>(Akk, lda, kb, k0, Linv + (size_t)b * NB * NB, ctx->d_info);
    GBEM_LAUNCH_CHECK(ctx);
    if (m > 0) {
      // L21 = A21 * inv(L11)^T  (in place, one CTA per 128-row strip)
      k_gemm_nt<kStore, 128><<<dim3((m + BM - 1) / BM, 1), GEMM_THREADS, Shape<128>::SMEM, s1>>>(
          A21, lda, A21, lda, Linv + (size_t)b * NB * NB, NB, m, kb, kb, 0, 0);
      GBEM_LAUNCH_CHECK(ctx);
    }
    GBEM_CUDA(ctx, cudaEventRecord(ctx->ev_panel, s1));
    GBEM_CUDA(ctx, cudaStreamWaitEvent(s, ctx->ev_panel, 0));
    if (m <= 0) break;
    // A22 -= L21 L21^T: first the next block column (tile column 0), then the rest
    int nt = (m + BM - 1) / BM;
    double* A22 = ctx->d_A + (long long)(k0 + kb) * lda + (k0 + kb);
    constexpr int kSplit = NB / 64;  // block column k+1 = kSplit tile columns of 64
    k_gemm_nt<kSub, 64><<<dim3(nt, kSplit), GEMM_THREADS, Shape<64>::SMEM, s>>>(A22, lda, A21, lda, A21, lda, m, m,
                                                                               kb, 2, kSplit);
    GBEM_LAUNCH_CHECK(ctx);
    GBEM_CUDA(ctx, cudaEventRecord(ctx->ev_col, s));
    if (nt > 1) {
      long long rest = lower_tiles_before<64>(nt) - (long long)kSplit * nt;
      k_gemm_nt<kSub, 64><<<(unsigned)rest, GEMM_THREADS, Shape<64>::SMEM, s>>>(A22, lda, A21, lda, A21, lda, m, m,
                                                                              kb, 3, kSplit);
      GBEM_LAUNCH_CHECK(ctx);
    }
  }
  cudaEventRecord(ctx->ev[1], s);
  GBEM_CUDA(ctx, cudaMemcpyAsync(ctx->h_info, ctx->d_info, sizeof(int), cudaMemcpyDeviceToHost, s));
  GBEM_CUDA(ctx, cudaStreamSynchronize(s));
  ctx->factored = true;
  if (*ctx->h_info != big) {
    if (stats) stats->bad_pivot = *ctx->h_info;
    return ctx->fail(GBEM_ENUMERIC,
                     "matrix not positive definite (pivot at row " + std::to_string(*ctx->h_info) + ")");
  }
  if (nrhs == 0) return GBEM_OK;
  // X <- B, then forward / backward substitution in place
  k_copy<<<(unsigned)(((long long)n * nrhs + 255) / 256), 256, 0, s>>>(d_B, d_X, (long long)n * nrhs);
  GBEM_LAUNCH_CHECK(ctx);
  const int R = (int)nrhs;
  for (int b = 0; b < nblk; ++b) {
    int k0 = b * NB, kb = std::min(NB, n - k0);
    k_trsv_diag<<<R, 128, 0, s>>>(Linv + (size_t)b * NB * NB, kb, d_X, n, k0, R, 0);
    GBEM_LAUNCH_CHECK(ctx);
    int m = n - k0 - kb;
    if (m > 0) {
      dim3 grid((m + 127) / 128);
      for (int q0 = 0; q0 < R; q0 += 32) {
        int rq = std::min(32, R - q0);
        double* Xq = d_X + (long long)q0 * n;
        if (rq <= 8)
          k_fwd_update<8><<<grid, 128, 0, s>>>(ctx->d_A, lda, k0, kb, n, Xq, n, rq);
        else if (rq <= 16)
          k_fwd_update<16><<<grid, 128, 0, s>>>(ctx->d_A, lda, k0, kb, n, Xq, n, rq);
        else
          k_fwd_update<32><<<grid, 128, 0, s>>>(ctx->d_A, lda, k0, kb, n, Xq, n, rq);
        GBEM_LAUNCH_CHECK(ctx);
      }
    }
  }
  for (int b = nblk - 1; b >= 0; --b) {
    int k0 = b * NB, kb = std::min(NB, n - k0);
    k_trsv_diag<<<R, 128, 0, s>>>(Linv + (size_t)b * NB * NB, kb, d_X, n, k0, R, 1);
    GBEM_LAUNCH_CHECK(ctx);
    if (k0 > 0) {
      dim3 grid((k0 + 7) / 8);
      for (int q0 = 0; q0 < R; q0 += 32) {
        int rq = std::min(32, R - q0);
        double* Xq = d_X + (long long)q0 * n;
        if (rq <= 8)
          k_bwd_update<8><<<grid, 256, 0, s>>>(ctx->d_A, lda, k0, kb, Xq, n, rq);
        else if (rq <= 16)
          k_bwd_update<16><<<grid, 256, 0, s>>>(ctx->d_A, lda, k0, kb, Xq, n, rq);
        else
          k_bwd_update<32><<<grid, 256, 0, s>>>(ctx->d_A, lda, k0, kb, Xq, n, rq);
        GBEM_LAUNCH_CHECK(ctx);
      }
    }
  }
  cudaEventRecord(ctx->ev[2], s);
  if (d_resid) {
    GBEM_CUDA(ctx, cudaMemsetAsync(Ysym, 0, sizeof(double) * (size_t)n * R, s));
    int nbt = (n + 63) / 64;
    long long ntiles = (long long)nbt * (nbt + 1) / 2;
    for (int q0 = 0; q0 < R; q0 += 32) {
      int rq = std::min(32, R - q0);
      const double* Xq = d_X + (long long)q0 * n;
      double* Yq = Ysym + (long long)q0 * n;
      if (rq <= 8)
        k_symv_upper<8><<<(unsigned)ntiles, 128, 0, s>>>(ctx->d_A, lda, ctx->d_diag, n, Xq, n, rq, Yq);
      else if (rq <= 16)
        k_symv_upper<16><<<(unsigned)ntiles, 128, 0, s>>>(ctx->d_A, lda, ctx->d_diag, n, Xq, n, rq, Yq);
      else
        k_symv_upper<32><<<(unsigned)ntiles, 128, 0, s>>>(ctx->d_A, lda, ctx->d_diag, n, Xq, n, rq, Yq);
      GBEM_LAUNCH_CHECK(ctx);
    }
    k_resid_norm<<<R, 256, 0, s>>>(Ysym, d_B, n, d_resid);
    GBEM_LAUNCH_CHECK(ctx);
  }
  cudaEventRecord(ctx->ev[3], s);
  if (stats) {
    GBEM_CUDA(ctx, cudaEventSynchronize(ctx->ev[3]));
    float a = 0, b2 = 0, c = 0;
    cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]);
    cudaEventElapsedTime(&b2, ctx->ev[1], ctx->ev[2]);
    cudaEventElapsedTime(&c, ctx->ev[2], ctx->ev[3]);
    stats->ms_factor = a;
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

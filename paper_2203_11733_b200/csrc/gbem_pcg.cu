// gbem_pcg.cu — row-block sharded C-matrix extraction: block-Jacobi
// preconditioned CG over NCCL (or host-provided collectives), all on the device.
//
// SURVEY.md §8b/§8e.  The reference has no iterative or distributed solver
// (solver.hpp:24-50 is dense Cholesky); this path reproduces what the direct
// path feeds into net_charges (extraction.hpp:55-79) when A does not fit one
// GPU.  Rank r of P owns complete rows [r m, min((r+1) m, n)), m = ceil(n / P),
// stored COLUMN-major (m x n, ld mA): the row-block product Q = A_r P is then
// the NT DMMA GEMM  Q^T (Kp x m) = P_full^T (Kp x n) * (A_r (m x n))^T  with
// P_full row-major (n x Kp, the all-gathered search directions) — the same
// memory reads as a row-major A_r, in the layout the tensor-core GEMM takes.
// All CG vectors are row-major m x Kp (Kp = K rounded up to 8; padded columns
// start converged), so a rank's search-direction slot is one contiguous
// all-gather contribution.
//
// Per iteration (one stream, no host synchronisation inside an iteration):
//   all_gather(P_r -> P_full)                          NCCL / host collective
//   Qpart_s = split-K slices of P_full^T A_r^T         k_gemm_nt_sk (DMMA)
//   Q = sum_s Qpart_s ; pq += P.Q                      k_sum_dot
//   all_reduce(pq)
//   alpha = rz / pq  (active columns)                  k_alpha
//   X += alpha P ; R -= alpha Q                        k_update_xr
//   Zpart = R^T Minv_b per Jacobi block                k_gemm_nt_sk (DMMA)
//   Z = sum_s Zpart ; rr += R.R ; rzn += R.Z           k_sum_dot2
//   all_reduce(rr, rzn)
//   active, beta, rz ; done flag                       k_beta
//   P = Z + beta P                                     k_update_p
// The host reads the done flag of iteration i-1 after enqueueing iteration i
// (the device always has an iteration queued; a finished run executes one
// extra iteration with every column frozen, alpha = beta = 0).  Afterwards the
// true residual ||B - A X|| / ||B|| is recomputed from A (solver.hpp:47) and the
// charges are reduced per rank and all-reduced.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "gbem_ctx.cuh"
#include "gbem_dmma_gemm.cuh"
#include "gbem_gemm_sk.cuh"

namespace {

using gbem_gemm::BK;
using gbem_sk::k_gemm_nt_sk;
using gbem_sk::k_gemm_nt_sk_bulk;
using gbem_sk::kSmem;
using gbem_sk::kT;
using gbem_sk::kThreads;

// ---------------------------------------------------------------- NCCL, loaded at run time
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // the soname first: a process that already mapped NCCL (torch) shares that copy
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
    api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.AllReduce &&
             api.GetErrorString;
    if (!api.ok) api.err = "libnccl.so.2 lacks an expected symbol";
  });
  return api;
}

#define GBEM_NCCL(ctx, call)                                                                       \
  do {                                                                                             \
    ncclResult_t r_ = (call);                                                                      \
    if (r_ != ncclSuccess)                                                                         \
      return (ctx)->fail(GBEM_ECUDA, std::string(#call) + ": " + nccl().GetErrorString(r_));       \
  } while (0)

int coll_all_gather(gbem_ctx* ctx, const double* send, double* recv, int64_t count) {
  if (ctx->nranks == 1) {
    if (send != recv)
      GBEM_CUDA(ctx, cudaMemcpyAsync(recv, send, sizeof(double) * count, cudaMemcpyDeviceToDevice, ctx->stream));
    return GBEM_OK;
  }
  if (ctx->nccl_comm)
    GBEM_NCCL(ctx, nccl().AllGather(send, recv, (size_t)count, ncclFloat64, (ncclComm_t)ctx->nccl_comm, ctx->stream));
  else if (ctx->has_coll) {
    if (ctx->coll.all_gather(ctx->coll.user, send, recv, count, ctx->stream))
      return ctx->fail(GBEM_ECUDA, "host all_gather collective failed");
  } else
    return ctx->fail(GBEM_EINVAL, "no collectives attached for nranks > 1");
  return GBEM_OK;
}

int coll_all_reduce(gbem_ctx* ctx, double* buf, int64_t count) {
  if (ctx->nranks == 1) return GBEM_OK;
  if (ctx->nccl_comm)
    GBEM_NCCL(ctx, nccl().AllReduce(buf, buf, (size_t)count, ncclFloat64, ncclSum, (ncclComm_t)ctx->nccl_comm,
                                    ctx->stream));
  else if (ctx->has_coll) {
    if (ctx->coll.all_reduce_sum(ctx->coll.user, buf, count, ctx->stream))
      return ctx->fail(GBEM_ECUDA, "host all_reduce collective failed");
  } else
    return ctx->fail(GBEM_EINVAL, "no collectives attached for nranks > 1");
  return GBEM_OK;
}

// ---------------------------------------------------------------- CG vector kernels
// Vectors are row-major rows x Kp.  A thread keeps one column k = gid % Kp and
// strides by T = (grid threads rounded down to a multiple of Kp), so its dot
// partials belong to one column; a CTA folds them in shared memory and adds
// one atomic per column.
enum Slot { S_PQ = 0, S_RR, S_RZN, S_BB, S_RZ, S_ALPHA, S_BETA, S_ACTIVE, S_REL, S_COUNT };

__device__ __forceinline__ long long grid_stride_cols(int Kp) {
  const long long t = (long long)gridDim.x * blockDim.x;
  return t - t % Kp;
}

// Q = sum_s Qp[s] (rows x Kp each, stride sstride); dot[k] += sum_i P(i,k) Q(i,k)
__global__ void k_sum_dot(const double* __restrict__ Qp, long long sstride, int S, double* __restrict__ Q,
                          const double* __restrict__ Pv, long long cnt, int Kp, double* dot) {
  extern __shared__ double red[];  // [Kp]
  for (int k = threadIdx.x; k < Kp; k += blockDim.x) red[k] = 0.0;
  __syncthreads();
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x, T = grid_stride_cols(Kp);
  if (gid < T) {
    double acc = 0.0;
    for (long long e = gid; e < cnt; e += T) {
      double q = Qp[e];
      for (int s = 1; s < S; ++s) q += Qp[s * sstride + e];
      Q[e] = q;
      acc = fma(Pv[e], q, acc);
    }
    atomicAdd(&red[gid % Kp], acc);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < Kp; k += blockDim.x) atomicAdd(&dot[k], red[k]);
}

// Z = sum_s Zp[s]; rr[k] += R.R, rzn[k] += R.Z   (dots: rr at dots[0..Kp), rzn at dots[Kp..2Kp))
__global__ void k_sum_dot2(const double* __restrict__ Zp, long long sstride, int S, double* __restrict__ Z,
                           const double* __restrict__ R, long long cnt, int Kp, double* dots) {
  extern __shared__ double red[];  // [2 Kp]
  for (int k = threadIdx.x; k < 2 * Kp; k += blockDim.x) red[k] = 0.0;
  __syncthreads();
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x, T = grid_stride_cols(Kp);
  if (gid < T) {
    double rr = 0.0, rz = 0.0;
    for (long long e = gid; e < cnt; e += T) {
      double z = Zp[e];
      for (int s = 1; s < S; ++s) z += Zp[s * sstride + e];
      Z[e] = z;
      const double r = R[e];
      rr = fma(r, r, rr);
      rz = fma(r, z, rz);
    }
    atomicAdd(&red[gid % Kp], rr);
    atomicAdd(&red[Kp + gid % Kp], rz);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 2 * Kp; k += blockDim.x) atomicAdd(&dots[k], red[k]);
}

// rres[k] += (B - sum_s Qp[s])^2 (true residual of the final X)
__global__ void k_resid_dot(const double* __restrict__ Qp, long long sstride, int S, const double* __restrict__ B,
                            long long cnt, int Kp, double* dot) {
  extern __shared__ double red[];
  for (int k = threadIdx.x; k < Kp; k += blockDim.x) red[k] = 0.0;
  __syncthreads();
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x, T = grid_stride_cols(Kp);
  if (gid < T) {
    double acc = 0.0;
    for (long long e = gid; e < cnt; e += T) {
      double q = Qp[e];
      for (int s = 1; s < S; ++s) q += Qp[s * sstride + e];
      const double d = B[e] - q;
      acc = fma(d, d, acc);
    }
    atomicAdd(&red[gid % Kp], acc);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < Kp; k += blockDim.x) atomicAdd(&dot[k], red[k]);
}

// B(i, k) = [net(row_begin + i) == k]; X = 0; R = B; bb[k] += B.B (padded rows / columns stay 0)
__global__ void k_init_rhs(const int32_t* __restrict__ net, long long row_begin, long long rows, int K, int Kp,
                           long long cnt, double* B, double* X, double* R) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / Kp;
    const int k = (int)(e % Kp);
    const double b = (i < rows && k < K && net[row_begin + i] == k) ? 1.0 : 0.0;
    B[e] = b;
    R[e] = b;
    X[e] = 0.0;
  }
}

// after the first preconditioner application: rz = rzn; active = bb > 0 and
// sqrt(rr / bb) > tol; rel; zero the accumulators
__global__ void k_start(double* sc, int Kp, double tol, int* done) {
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  for (int k = threadIdx.x; k < Kp; k += blockDim.x) {
    const double bb = sc[S_BB * Kp + k], rr = sc[S_RR * Kp + k];
    const double rel = bb > 0.0 ? sqrt(rr / bb) : 0.0;
    const bool act = bb > 0.0 && rel > tol;
    sc[S_RZ * Kp + k] = sc[S_RZN * Kp + k];
    sc[S_ACTIVE * Kp + k] = act ? 1.0 : 0.0;
    sc[S_REL * Kp + k] = rel;
    sc[S_PQ * Kp + k] = sc[S_RR * Kp + k] = sc[S_RZN * Kp + k] = 0.0;
    if (act) any = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) *done = any ? 0 : 1;
}

__global__ void k_alpha(double* sc, int Kp) {
  for (int k = threadIdx.x; k < Kp; k += blockDim.x) {
    const double pq = sc[S_PQ * Kp + k];
    sc[S_ALPHA * Kp + k] = (sc[S_ACTIVE * Kp + k] != 0.0 && pq > 0.0) ? sc[S_RZ * Kp + k] / pq : 0.0;
    sc[S_PQ * Kp + k] = 0.0;
  }
}

__global__ void k_update_xr(const double* __restrict__ sc, int Kp, long long cnt, const double* __restrict__ Pv,
                            const double* __restrict__ Q, double* X, double* R) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += (long long)gridDim.x * blockDim.x) {
    const double a = sc[S_ALPHA * Kp + (int)(e % Kp)];
    X[e] = fma(a, Pv[e], X[e]);
    R[e] = fma(-a, Q[e], R[e]);
  }
}

__global__ void k_beta(double* sc, int Kp, double tol, int* done) {
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  for (int k = threadIdx.x; k < Kp; k += blockDim.x) {
    const double bb = sc[S_BB * Kp + k], rr = sc[S_RR * Kp + k], rzn = sc[S_RZN * Kp + k];
    bool act = sc[S_ACTIVE * Kp + k] != 0.0;
    if (act) {
      const double rel = sqrt(rr / bb);
      sc[S_REL * Kp + k] = rel;
      act = rel > tol;
    }
    const double rz = sc[S_RZ * Kp + k];
    sc[S_BETA * Kp + k] = act && rz != 0.0 ? rzn / rz : 0.0;
    if (act) sc[S_RZ * Kp + k] = rzn;
    sc[S_ACTIVE * Kp + k] = act ? 1.0 : 0.0;
    sc[S_RR * Kp + k] = sc[S_RZN * Kp + k] = 0.0;
    if (act) any = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) *done = any ? 0 : 1;
}

__global__ void k_update_p(const double* __restrict__ sc, int Kp, long long cnt, const double* __restrict__ Z,
                           double* Pv) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(e % Kp);
    if (sc[S_ACTIVE * Kp + k] != 0.0) Pv[e] = fma(sc[S_BETA * Kp + k], Pv[e], Z[e]);
  }
}

__global__ void k_copy(const double* __restrict__ src, double* __restrict__ dst, long long cnt) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += (long long)gridDim.x * blockDim.x)
    dst[e] = src[e];
}

__global__ void k_identity(double* I, long long m) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m * m; e += (long long)gridDim.x * blockDim.x)
    I[e] = (e / m == e % m) ? 1.0 : 0.0;
}

// ---- explicit inverse of a factored Jacobi block from its Cholesky factor (n^3 flops instead of
// the 2.3 n^3 of two dense triangular solves against the identity):
//   N = -inv(L)^T (upper) and Y = N^T (lower) are built bottom-up over groups of 128-row blocks,
//   [[L11, 0], [L21, L22]] -> N12 = N11 L21^T N22 (two NT GEMMs: T = N11 L21^T, N12 = T Y22^T; the
//   signs cancel; each skips the zero half of its triangular operand), Y21 = N12^T; the 128 x 128 base blocks come from the factorisation's own
//   inverses of its diagonal blocks; then inv(M) = N N^T (k_syrk_bulk<TRI_STORE>, the reduction of a
//   tile starting at its first non-zero column) and a mirror into the upper triangle.
constexpr int kInvNB = 128;

__global__ void __launch_bounds__(256)
    k_inv_base(const double* __restrict__ Linv, int n, double* Nm, double* Ym, long long ld) {
  const int b = blockIdx.x, r0 = b * kInvNB;
  for (int idx = threadIdx.x; idx < kInvNB * kInvNB; idx += blockDim.x) {
    const int c = idx / kInvNB, r = idx % kInvNB;
    if (r0 + r < n && r0 + c < n && r >= c) {
      const double v = -Linv[(size_t)b * kInvNB * kInvNB + c * kInvNB + r];  // inv(L_bb)(r, c)
      Ym[(long long)(r0 + c) * ld + r0 + r] = v;
      Nm[(long long)(r0 + r) * ld + r0 + c] = v;
    }
  }
}

// dst(j, i) = src(i, j), src rows x cols (column-major, lds), 32 x 32 tiles through shared memory
__global__ void __launch_bounds__(256)
    k_transpose(const double* __restrict__ src, long long lds, double* __restrict__ dst, long long ldd, int rows,
                int cols) {
  __shared__ double t[32][33];
  const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int jj = ty; jj < 32; jj += 8)
    if (i0 + tx < rows && j0 + jj < cols) t[jj][tx] = src[(long long)(j0 + jj) * lds + i0 + tx];
  __syncthreads();
  for (int ii = ty; ii < 32; ii += 8)
    if (j0 + tx < cols && i0 + ii < rows) dst[(long long)(i0 + ii) * ldd + j0 + tx] = t[tx][ii];
}

// A(c, r) = A(r, c) for r > c (lower triangle mirrored into the upper), n x n column-major
__global__ void __launch_bounds__(256) k_mirror_lower(double* A, long long ld, int n) {
  __shared__ double t[32][33];
  const int bi = blockIdx.x, bj = blockIdx.y;  // tile rows bi >= tile columns bj
  if (bj > bi) return;
  const int i0 = bi * 32, j0 = bj * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int jj = ty; jj < 32; jj += 8)
    if (i0 + tx < n && j0 + jj < n) t[jj][tx] = A[(long long)(j0 + jj) * ld + i0 + tx];
  __syncthreads();
  for (int ii = ty; ii < 32; ii += 8) {
    const int r = j0 + tx, c = i0 + ii;  // destination (row r, column c) = source (row c, column r)
    if (r < n && c < n && c > r) A[(long long)c * ld + r] = t[tx][ii];
  }
}

// Ct[r * K + k] += scale * X(i, r) for the local rows i with net(row_begin + i) = k;
// panels with net -1 (grounded outer panels) add to the outer charge Ct[K * K + r]
// (net_charges, extraction.hpp:55-79)
__global__ void k_rank_charges(const int32_t* __restrict__ net, long long row_begin, long long rows, int K, int Kp,
                               const double* __restrict__ X, double scale, double* Ct) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < rows * K; e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / K;
    const int r = (int)(e % K);
    const int k = net[row_begin + i];
    if (k >= 0 && k < K)
      atomicAdd(&Ct[(long long)r * K + k], scale * X[i * Kp + r]);
    else
      atomicAdd(&Ct[(long long)K * K + r], scale * X[i * Kp + r]);
  }
}

__global__ void k_finish_resid(const double* sc_rres, const double* sc, int K, int Kp, double* resid) {
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    const double bb = sc[S_BB * Kp + k];
    resid[k] = bb > 0.0 ? sqrt(sc_rres[k] / bb) : 0.0;
  }
}

// ---------------------------------------------------------------- workspace
struct Ws {
  size_t cap_A = 0, cap_vec = 0, cap_full = 0, cap_part = 0, cap_minv = 0, cap_tmp = 0, cap_inv = 0;
  double* A = nullptr;      // m x n column-major rows of this rank (ld mA)
  double* vec = nullptr;    // B, X, R, Z, P, Q : 6 x (m Kp)
  double* full = nullptr;   // P_full: nranks m x Kp
  double* part = nullptr;   // split-K partials
  double* minv = nullptr;   // explicit inverses of the Jacobi blocks
  double* tmp = nullptr;    // identity for the inverse solves
  double* inv = nullptr;    // N, Y, T of the GEMM-form block inverse
  double* sc = nullptr;     // scalars: S_COUNT x Kp, then rres (Kp), then C (K x K)
  size_t cap_sc = 0;
  int* d_done = nullptr;
  int* h_done = nullptr;    // pinned, two slots
  std::vector<cudaEvent_t> ev;
};

void release(gbem_ctx* ctx) {
  Ws* w = (Ws*)ctx->pcg_ws;
  if (w) {
    cudaFree(w->A);
    cudaFree(w->vec);
    cudaFree(w->full);
    cudaFree(w->part);
    cudaFree(w->minv);
    cudaFree(w->tmp);
    cudaFree(w->inv);
    cudaFree(w->sc);
    cudaFree(w->d_done);
    if (w->h_done) cudaFreeHost(w->h_done);
    for (auto e : w->ev) cudaEventDestroy(e);
    delete w;
    ctx->pcg_ws = nullptr;
  }
  if (ctx->nccl_comm && nccl().ok) nccl().CommDestroy((ncclComm_t)ctx->nccl_comm);
  ctx->nccl_comm = nullptr;
}

Ws* ws(gbem_ctx* ctx) {
  if (!ctx->pcg_ws) {
    ctx->pcg_ws = new Ws();
    ctx->pcg_release = release;
  }
  return (Ws*)ctx->pcg_ws;
}

int grow(gbem_ctx* ctx, double** p, size_t* cap, size_t need) {
  if (*cap >= need && *p) return GBEM_OK;
  cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  GBEM_CUDA(ctx, cudaMalloc(p, std::max<size_t>(need, 1) * sizeof(double)));
  *cap = need;
  return GBEM_OK;
}

int ensure_gemm_attrs(gbem_ctx* ctx) {
  if (!(ctx->attr_set & gbem_ctx::kAttrPcgGemm)) {
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_gemm_nt_sk<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_gemm_nt_sk_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)gbem_sk::SkBulk::SMEM));
    GBEM_CUDA(ctx, cudaFuncSetAttribute(gbem_gemm::k_syrk_bulk<16, 3, 4, true, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gbem_sk::SkBulk::SMEM));
    ctx->attr_set |= gbem_ctx::kAttrPcgGemm;
  }
  return GBEM_OK;
}

// Explicit inverse of the Jacobi block whose Cholesky factor is in ctx->d_A (mb x mb, the
// factorisation's diagonal-block inverses in ctx->d_linv) into out (column-major, ld = mb); see the
// kernels above.  `ws` holds N, Y (ld x ld each, ld = mb rounded up to 16) and T.
int block_inverse_gemm(gbem_ctx* ctx, double* ws, long long mb, double* out) {
  cudaStream_t s = ctx->stream;
  if (int rc = ensure_gemm_attrs(ctx)) return rc;
  const long long ld = (mb + 15) / 16 * 16;
  double *Nm = ws, *Ym = ws + ld * ld, *T = Ym + ld * ld;
  GBEM_CUDA(ctx, cudaMemsetAsync(Nm, 0, sizeof(double) * 2 * (size_t)(ld * ld), s));
  const int nblk = (int)((mb + kInvNB - 1) / kInvNB);
  k_inv_base<<<nblk, 256, 0, s>>>(ctx->d_linv, (int)mb, Nm, Ym, ld);
  GBEM_LAUNCH_CHECK(ctx);
  auto gemm_store = [&](double* C, long long ldc, const double* A, long long lda, const double* B, long long ldb, int M,
                        int N, int K, int tri) -> int {
    const long long kchunk = ((long long)K + BK - 1) / BK * BK;
    dim3 grid((unsigned)((M + kT - 1) / kT), (unsigned)((N + kT - 1) / kT), 1);
    k_gemm_nt_sk_bulk<<<grid, 128, gbem_sk::SkBulk::SMEM, s>>>(C, ldc, 0, A, lda, B, ldb, M, N, K, kchunk, tri);
    GBEM_LAUNCH_CHECK(ctx);
    return GBEM_OK;
  };
  const long long lda = ctx->lda;
  for (int len = 1; len < nblk; len *= 2)
    for (int g = 0; g + len < nblk; g += 2 * len) {
      const long long r0 = (long long)g * kInvNB, r1 = (long long)(g + len) * kInvNB;
      const long long r2 = std::min<long long>((long long)(g + 2 * len) * kInvNB, mb);
      const int s1 = (int)(r1 - r0), s2 = (int)(r2 - r1);
      // T = N11 L21^T (s1 x s2), then N12 = T Y22^T, then Y21 = N12^T
      if (int rc = gemm_store(T, s1, Nm + r0 * ld + r0, ld, ctx->d_A + r0 * lda + r1, lda, s1, s2, s1, 1)) return rc;
      if (int rc = gemm_store(Nm + r1 * ld + r0, ld, T, s1, Ym + r1 * ld + r1, ld, s1, s2, s2, 2)) return rc;
      k_transpose<<<dim3((unsigned)((s1 + 31) / 32), (unsigned)((s2 + 31) / 32)), 256, 0, s>>>(
          Nm + r1 * ld + r0, ld, Ym + r0 * ld + r1, ld, s1, s2);
      GBEM_LAUNCH_CHECK(ctx);
    }
  const long long nt = (mb + 63) / 64;
  gbem_gemm::k_syrk_bulk<16, 3, 4, true, true><<<(unsigned)(nt * (nt + 1) / 2), 128, gbem_sk::SkBulk::SMEM, s>>>(
      out, mb, Nm, ld, (int)mb, (int)ld, 0, 0, nullptr);
  GBEM_LAUNCH_CHECK(ctx);
  const unsigned n32 = (unsigned)((mb + 31) / 32);
  k_mirror_lower<<<dim3(n32, n32), 256, 0, s>>>(out, mb, (int)mb);
  GBEM_LAUNCH_CHECK(ctx);
  return GBEM_OK;
}

// C_z = A * B^T split over `S` slices of Ktot (Kp rows of C handled in 64-row chunks)
int gemm_nt(gbem_ctx* ctx, double* C, long long ldc, long long strideC, const double* A, long long lda,
            const double* B, long long ldb, int M, int N, long long Ktot, int S) {
  static_assert(kSmem <= 227 * 1024, "smem");
  if (int rc = ensure_gemm_attrs(ctx)) return rc;
  static const bool use_bulk = getenv("GBEM_PCG_CPASYNC") == nullptr;
  long long kchunk = (Ktot + S - 1) / S;
  kchunk = (kchunk + BK - 1) / BK * BK;
  const int vec16 = (lda % 2 == 0 && ldb % 2 == 0 && ((uintptr_t)A & 15) == 0 && ((uintptr_t)B & 15) == 0) ? 1 : 0;
  for (int m0 = 0; m0 < M; m0 += kT) {
    const int mm = std::min(kT, M - m0);
    dim3 grid(1, (unsigned)((N + kT - 1) / kT), (unsigned)S);
    // bulk-copy staging: 16-byte copies rounded up from an odd row count must stay inside the column
    const bool bulk = use_bulk && vec16 && (mm % 2 == 0 || m0 + mm < lda) && (N % 2 == 0 || N < ldb);
    if (bulk)
      k_gemm_nt_sk_bulk<<<grid, 128, gbem_sk::SkBulk::SMEM, ctx->stream>>>(C + m0, ldc, strideC, A + m0, lda, B, ldb,
                                                                          mm, N, Ktot, kchunk);
    else
      k_gemm_nt_sk<64><<<grid, kThreads, kSmem, ctx->stream>>>(C + m0, ldc, strideC, A + m0, lda, B, ldb, mm, N,
                                                              Ktot, kchunk, vec16 && (m0 % 2 == 0));
    GBEM_LAUNCH_CHECK(ctx);
  }
  return GBEM_OK;
}

// Split count of the reduction dimension: at least ~2.2 waves of CTAs (a
// single partial wave leaves SMs with unequal CTA counts) and at least 4 slices
// of a large product (a shorter tail wave), each slice >= 32 BK steps.
// tools/pcg_gemm_bench.cu at Kp = 64, n = 96,200: rows 12,032 -> S = 7
// (30.2 TFLOP/s vs 27.4 at S = 3); rows 96,200 -> S = 4 (31.8 vs 28.7 at S = 1).
int splits_for(gbem_ctx* ctx, long long tiles, long long Ktot) {
  const long long slots = 4LL * ctx->num_sms;
  tiles = std::max<long long>(1, tiles);
  const long long target = std::max<long long>(22 * slots / 10, 4 * tiles);
  long long s = (target + tiles - 1) / tiles;
  // bulk-staged kernel, tools/pcg_gemm_bench.cu at Kp = 64, n = 96,200 (TFLOP/s at S = 4 / 7):
  // 12,025 rows 29.9 / 34.7, 24,050 rows 32.4 / 35.0, 48,100 rows 34.5 / 35.5, 96,200 rows 35.6 / 35.6
  if (tiles >= 150 && s < 7) s = 7;
  s = std::min<long long>(s, std::max<long long>(1, Ktot / 512));
  return (int)std::max<long long>(1, std::min<long long>(s, 8));
}

}  // namespace

extern "C" {

int gbem_nccl_unique_id(void* id_out) {
  if (!id_out) return GBEM_EINVAL;
  const NcclApi& a = nccl();
  if (!a.ok) return GBEM_ECUDA;
  ncclUniqueId id;
  if (a.GetUniqueId(&id) != ncclSuccess) return GBEM_ECUDA;
  static_assert(sizeof(ncclUniqueId) == GBEM_NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");
  memcpy(id_out, &id, sizeof(id));
  return GBEM_OK;
}

int gbem_ctx_init_nccl(gbem_ctx* ctx, int32_t nranks, int32_t rank, const void* id) {
  if (!ctx) return GBEM_EINVAL;
  if (nranks < 1 || rank < 0 || rank >= nranks || !id) return ctx->fail(GBEM_EINVAL, "bad nranks / rank / id");
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  const NcclApi& a = nccl();
  if (!a.ok) return ctx->fail(GBEM_ECUDA, a.err);
  if (ctx->nccl_comm) {
    a.CommDestroy((ncclComm_t)ctx->nccl_comm);
    ctx->nccl_comm = nullptr;
  }
  ws(ctx);  // registers the release hook
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm;
  GBEM_NCCL(ctx, a.CommInitRank(&comm, nranks, uid, rank));
  ctx->nccl_comm = comm;
  ctx->nranks = nranks;
  ctx->rank = rank;
  ctx->has_coll = false;
  return GBEM_OK;
}

int gbem_ctx_set_collectives(gbem_ctx* ctx, int32_t nranks, int32_t rank, const gbem_collectives* coll) {
  if (!ctx) return GBEM_EINVAL;
  if (nranks < 1 || rank < 0 || rank >= nranks) return ctx->fail(GBEM_EINVAL, "bad nranks / rank");
  if (nranks > 1 && (!coll || !coll->all_gather || !coll->all_reduce_sum))
    return ctx->fail(GBEM_EINVAL, "collectives required for nranks > 1");
  ws(ctx);
  if (ctx->nccl_comm && nccl().ok) nccl().CommDestroy((ncclComm_t)ctx->nccl_comm);
  ctx->nccl_comm = nullptr;
  ctx->nranks = nranks;
  ctx->rank = rank;
  ctx->has_coll = nranks > 1;
  if (coll) ctx->coll = *coll;
  return GBEM_OK;
}

}  // extern "C"

namespace {

int pcg_extract(gbem_ctx* ctx, const gbem_panels* P, bool device_panels, int64_t n, const int32_t* net, int32_t K,
                double eps_r, const gbem_quad_config* cfg, const gbem_pcg_options* opt_in, double* C_out,
                double* resid_out, double* outer_out, gbem_assembly_stats* astats, gbem_pcg_stats* pstats) {
  gbem_pcg_options opt{1e-10, 1000, 1};
  if (opt_in) {
    if (opt_in->tol > 0) opt.tol = opt_in->tol;
    if (opt_in->max_iter > 0) opt.max_iter = opt_in->max_iter;
    if (opt_in->jacobi_blocks > 0) opt.jacobi_blocks = opt_in->jacobi_blocks;
  }
  Ws* w = ws(ctx);
  cudaStream_t s = ctx->stream;
  const int R = ctx->nranks, rank = ctx->rank;
  const long long m = (n + R - 1) / R;
  const long long rb = std::min<long long>(n, (long long)rank * m);
  const long long rows = std::min<long long>(n, rb + m) - rb;
  const long long mA = (m + 7) / 8 * 8;
  const int Kp = (K + 7) / 8 * 8;
  const long long cnt = m * Kp;      // local vector slot (all-gather contribution)
  const long long cntr = rows * Kp;  // its live part: padded rows stay zero
  if (w->ev.empty()) {
    w->ev.resize(8);
    for (auto& e : w->ev) GBEM_CUDA(ctx, cudaEventCreate(&e));
  }
  if (!w->d_done) {
    GBEM_CUDA(ctx, cudaMalloc(&w->d_done, sizeof(int)));
    GBEM_CUDA(ctx, cudaMallocHost(&w->h_done, 2 * sizeof(int)));
  }
  int rc;
  // --- 1. assembly of complete rows, no communication (column-major m x n)
  rc = grow(ctx, &w->A, &w->cap_A, (size_t)mA * (size_t)n);
  if (rc) return rc;
  rc = gbem_internal_upload_panels(ctx, P, n, device_panels);
  if (rc) return rc;
  cudaEventRecord(w->ev[0], s);
  if (rows > 0) {
    rc = gbem_internal_assemble(ctx, n, rb, rb + rows, cfg, astats, false, w->A, mA, true, true);
    if (rc) return rc;
  }
  cudaEventRecord(w->ev[1], s);
  // --- 2. block-Jacobi preconditioner: explicit inverse of each diagonal block
  const int nb = (int)std::max<long long>(1, std::min<long long>(opt.jacobi_blocks, std::max<long long>(rows, 1)));
  std::vector<long long> cut(nb + 1), moff(nb + 1, 0);
  for (int b = 0; b <= nb; ++b) cut[b] = b == nb ? rows : rows * b / nb / 8 * 8;  // 8-row aligned blocks
  for (int b = 0; b < nb; ++b) moff[b + 1] = moff[b] + (cut[b + 1] - cut[b]) * (cut[b + 1] - cut[b]);
  rc = grow(ctx, &w->minv, &w->cap_minv, (size_t)std::max<long long>(moff[nb], 1));
  if (rc) return rc;
  long long mbmax = 0;
  for (int b = 0; b < nb; ++b) mbmax = std::max(mbmax, cut[b + 1] - cut[b]);
  // GEMM-form inverse (N, Y, T: 2.25 ld^2 doubles) unless the block is too large for its workspace
  static const bool inv_solve_env = getenv("GBEM_PCG_INVERSE_BY_SOLVE") != nullptr;
  const long long ldi = (mbmax + 15) / 16 * 16;
  const bool inv_gemm = !inv_solve_env && mbmax >= 2 * kInvNB && mbmax <= 36000;
  if (inv_gemm)
    rc = grow(ctx, &w->inv, &w->cap_inv, (size_t)(2 * ldi * ldi + ldi * ldi / 4 + ldi * kInvNB));
  else
    rc = grow(ctx, &w->tmp, &w->cap_tmp, (size_t)std::max<long long>(mbmax * mbmax, 1));
  if (rc) return rc;
  for (int b = 0; b < nb; ++b) {
    const long long c0 = cut[b], mb = cut[b + 1] - cut[b];
    if (mb == 0) continue;
    rc = gbem_internal_ensure_matrix(ctx, mb, 0);
    if (rc) return rc;
    GBEM_CUDA(ctx, cudaMemcpy2DAsync(ctx->d_A, sizeof(double) * ctx->lda, w->A + (rb + c0) * mA + c0,
                                     sizeof(double) * mA, sizeof(double) * mb, mb, cudaMemcpyDeviceToDevice, s));
    rc = gbem_internal_factor(ctx, nullptr);
    if (rc) return rc;
    if (inv_gemm && mb >= 2 * kInvNB) {
      rc = block_inverse_gemm(ctx, w->inv, mb, w->minv + moff[b]);
      if (rc) return rc;
      continue;
    }
    if (!w->tmp || w->cap_tmp < (size_t)(mb * mb)) {
      rc = grow(ctx, &w->tmp, &w->cap_tmp, (size_t)std::max<long long>(mb * mb, 1));
      if (rc) return rc;
    }
    k_identity<<<(unsigned)std::min<long long>((mb * mb + 255) / 256, 65535), 256, 0, s>>>(w->tmp, mb);
    GBEM_LAUNCH_CHECK(ctx);
    rc = gbem_internal_solve_factored(ctx, w->tmp, mb, w->minv + moff[b], nullptr, nullptr);
    if (rc) return rc;
  }
  cudaEventRecord(w->ev[2], s);
  // --- 3. CG state
  rc = grow(ctx, &w->vec, &w->cap_vec, 6 * (size_t)cnt);
  if (rc) return rc;
  double *vB = w->vec, *vX = vB + cnt, *vR = vX + cnt, *vZ = vR + cnt, *vP = vZ + cnt, *vQ = vP + cnt;
  rc = grow(ctx, &w->full, &w->cap_full, (size_t)R * (size_t)cnt);
  if (rc) return rc;
  const long long tiles_mv = (rows + kT - 1) / kT * ((Kp + kT - 1) / kT);
  const int S_mv = splits_for(ctx, tiles_mv, n);
  int S_pc = 1;
  for (int b = 0; b < nb; ++b) {
    const long long mb = cut[b + 1] - cut[b];
    S_pc = std::max(S_pc, splits_for(ctx, (mb + kT - 1) / kT * ((Kp + kT - 1) / kT), mb));
  }
  const int S_max = std::max(S_mv, S_pc);
  rc = grow(ctx, &w->part, &w->cap_part, (size_t)S_max * (size_t)cnt);
  if (rc) return rc;
  rc = grow(ctx, &w->sc, &w->cap_sc, (size_t)(S_COUNT + 1) * Kp + (size_t)K * K + K);
  if (rc) return rc;
  double* sc = w->sc;
  double* rres = sc + S_COUNT * Kp;
  double* Ct = rres + Kp;
  GBEM_CUDA(ctx, cudaMemsetAsync(sc, 0, sizeof(double) * ((size_t)(S_COUNT + 1) * Kp + (size_t)K * K + K), s));
  GBEM_CUDA(ctx, cudaMemsetAsync(vZ, 0, sizeof(double) * 3 * (size_t)cnt, s));  // Z, P, Q
  const unsigned vgrid = (unsigned)std::min<long long>((cnt + 255) / 256, 8LL * ctx->num_sms);
  const size_t red1 = sizeof(double) * Kp, red2 = 2 * red1;
  k_init_rhs<<<vgrid, 256, 0, s>>>(net, rb, rows, K, Kp, cnt, vB, vX, vR);
  GBEM_LAUNCH_CHECK(ctx);
  auto precond = [&]() -> int {  // Zpart = R^T Minv_b, then Z, rr, rzn
    for (int b = 0; b < nb; ++b) {
      const long long c0 = cut[b], mb = cut[b + 1] - cut[b];
      if (mb == 0) continue;
      int rc2 = gemm_nt(ctx, w->part + c0 * Kp, Kp, cnt, vR + c0 * Kp, Kp, w->minv + moff[b], mb, Kp, (int)mb, mb,
                        S_pc);
      if (rc2) return rc2;
    }
    k_sum_dot2<<<vgrid, 256, red2, s>>>(w->part, cnt, S_pc, vZ, vR, cntr, Kp, sc + S_RR * Kp);
    GBEM_LAUNCH_CHECK(ctx);
    return GBEM_OK;
  };
  auto matvec = [&](const double* local) -> int {  // part = split slices of (A_r * gathered(local))
    int rc2 = coll_all_gather(ctx, local, w->full, cnt);
    if (rc2) return rc2;
    if (rows == 0) {
      GBEM_CUDA(ctx, cudaMemsetAsync(w->part, 0, sizeof(double) * cnt * S_mv, s));
      return GBEM_OK;
    }
    return gemm_nt(ctx, w->part, Kp, cnt, w->full, Kp, w->A, mA, Kp, (int)rows, n, S_mv);
  };
  // bb = B.B (k_sum_dot with Qp = P = B; its Q output lands in vQ, overwritten
  // by the first product), then the first preconditioner application
  k_sum_dot<<<vgrid, 256, red1, s>>>(vB, cnt, 1, vQ, vB, cntr, Kp, sc + S_BB * Kp);
  GBEM_LAUNCH_CHECK(ctx);
  rc = precond();
  if (rc) return rc;
  rc = coll_all_reduce(ctx, sc + S_RR * Kp, 3 * Kp);  // rr, rzn, bb
  if (rc) return rc;
  k_start<<<1, 256, 0, s>>>(sc, Kp, opt.tol, w->d_done);
  GBEM_LAUNCH_CHECK(ctx);
  k_copy<<<vgrid, 256, 0, s>>>(vZ, vP, cntr);
  GBEM_LAUNCH_CHECK(ctx);
  GBEM_CUDA(ctx, cudaMemcpyAsync(&w->h_done[0], w->d_done, sizeof(int), cudaMemcpyDeviceToHost, s));
  cudaEventRecord(w->ev[3], s);
  GBEM_CUDA(ctx, cudaEventSynchronize(w->ev[3]));
  int iters = 0;
  bool converged = w->h_done[0] != 0;
  double mv_flops = 0.0;
  float ms_mv = 0.f;
  if (!converged) {
    for (int it = 1; it <= opt.max_iter; ++it) {
      const bool timed = it == 1;
      if (timed) cudaEventRecord(w->ev[6], s);
      rc = matvec(vP);
      if (rc) return rc;
      if (timed) cudaEventRecord(w->ev[7], s);
      mv_flops += 2.0 * rows * (double)n * Kp;
      k_sum_dot<<<vgrid, 256, red1, s>>>(w->part, cnt, S_mv, vQ, vP, cntr, Kp, sc + S_PQ * Kp);
      GBEM_LAUNCH_CHECK(ctx);
      rc = coll_all_reduce(ctx, sc + S_PQ * Kp, Kp);
      if (rc) return rc;
      k_alpha<<<1, 256, 0, s>>>(sc, Kp);
      GBEM_LAUNCH_CHECK(ctx);
      k_update_xr<<<vgrid, 256, 0, s>>>(sc, Kp, cntr, vP, vQ, vX, vR);
      GBEM_LAUNCH_CHECK(ctx);
      rc = precond();
      if (rc) return rc;
      rc = coll_all_reduce(ctx, sc + S_RR * Kp, 2 * Kp);
      if (rc) return rc;
      k_beta<<<1, 256, 0, s>>>(sc, Kp, opt.tol, w->d_done);
      GBEM_LAUNCH_CHECK(ctx);
      k_update_p<<<vgrid, 256, 0, s>>>(sc, Kp, cntr, vZ, vP);
      GBEM_LAUNCH_CHECK(ctx);
      GBEM_CUDA(ctx, cudaMemcpyAsync(&w->h_done[it & 1], w->d_done, sizeof(int), cudaMemcpyDeviceToHost, s));
      cudaEventRecord(w->ev[4 + (it & 1)], s);
      if (timed) {
        GBEM_CUDA(ctx, cudaEventSynchronize(w->ev[7]));
        cudaEventElapsedTime(&ms_mv, w->ev[6], w->ev[7]);
      }
      // read iteration it-1's flag while iteration it runs
      if (it >= 2) {
        GBEM_CUDA(ctx, cudaEventSynchronize(w->ev[4 + ((it - 1) & 1)]));
        if (w->h_done[(it - 1) & 1]) {
          iters = it - 1;
          converged = true;
          break;
        }
      }
      iters = it;
    }
    if (!converged) {
      GBEM_CUDA(ctx, cudaEventSynchronize(w->ev[4 + (iters & 1)]));
      converged = w->h_done[iters & 1] != 0;
    }
  }
  cudaEventRecord(w->ev[3], s);
  // --- 4. true residual from A (solver.hpp:47), charges (extraction.hpp:55-79)
  rc = matvec(vX);
  if (rc) return rc;
  k_resid_dot<<<vgrid, 256, red1, s>>>(w->part, cnt, S_mv, vB, cntr, Kp, rres);
  GBEM_LAUNCH_CHECK(ctx);
  rc = coll_all_reduce(ctx, rres, Kp);
  if (rc) return rc;
  if (rows > 0) {
    k_rank_charges<<<(unsigned)std::min<long long>((rows * K + 255) / 256, 8LL * ctx->num_sms), 256, 0, s>>>(
        net, rb, rows, K, Kp, vX, eps_r * 8.854187817e-12 * 1e-6, Ct);
    GBEM_LAUNCH_CHECK(ctx);
  }
  rc = coll_all_reduce(ctx, Ct, (int64_t)K * K + K);
  if (rc) return rc;
  GBEM_CUDA(ctx, cudaMemcpyAsync(C_out, Ct, sizeof(double) * K * K, cudaMemcpyDeviceToDevice, s));
  if (outer_out)
    GBEM_CUDA(ctx, cudaMemcpyAsync(outer_out, Ct + (size_t)K * K, sizeof(double) * K, cudaMemcpyDeviceToDevice, s));
  double* dres = resid_out;
  if (!dres) dres = rres;  // in place (Kp >= K)
  k_finish_resid<<<1, 256, 0, s>>>(rres, sc, K, Kp, dres);
  GBEM_LAUNCH_CHECK(ctx);
  cudaEventRecord(w->ev[7], s);
  GBEM_CUDA(ctx, cudaEventSynchronize(w->ev[7]));
  std::vector<double> hres(K);
  GBEM_CUDA(ctx, cudaMemcpy(hres.data(), dres, sizeof(double) * K, cudaMemcpyDeviceToHost));
  double mx = 0.0;
  for (double v : hres) mx = std::max(mx, v);
  if (pstats) {
    gbem_pcg_stats& st = *pstats;
    st = gbem_pcg_stats{};
    st.n = n;
    st.rows_local = rows;
    st.row_begin = rb;
    st.nranks = R;
    st.rank = rank;
    st.iterations = iters;
    st.converged = converged ? 1 : 0;
    st.max_rel_resid = mx;
    float a = 0;
    cudaEventElapsedTime(&a, w->ev[0], w->ev[1]);
    st.ms_assembly = a;
    cudaEventElapsedTime(&a, w->ev[1], w->ev[2]);
    st.ms_precond = a;
    cudaEventElapsedTime(&a, w->ev[2], w->ev[3]);
    st.ms_iterations = a;
    cudaEventElapsedTime(&a, w->ev[0], w->ev[7]);
    st.ms_total = a;
    st.ms_matvec = ms_mv;  // one product (the first iteration's), device time
    st.matvec_flops = 2.0 * rows * (double)n * Kp;
  }
  if (!converged)
    return ctx->fail(GBEM_ENUMERIC, "block-Jacobi CG did not reach tol " + std::to_string(opt.tol) + " in " +
                                        std::to_string(opt.max_iter) + " iterations");
  (void)mv_flops;
  return GBEM_OK;
}

}  // namespace

extern "C" {

int gbem_pcg_extract_cmatrix_dev(gbem_ctx* ctx, const gbem_panels* P, int64_t n, const int32_t* net, int32_t K,
                                 double eps_r, const gbem_quad_config* cfg, const gbem_pcg_options* opt,
                                 double* C, double* resid, double* outer, gbem_assembly_stats* astats,
                                 gbem_pcg_stats* pstats) {
  if (!ctx) return GBEM_EINVAL;
  if (!P || !net || !C || n <= 0) return ctx->fail(GBEM_EINVAL, "null argument or empty panel set");
  if (K < 1 || K > 2048) return ctx->fail(GBEM_EINVAL, "K must be in [1, 2048]");
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  return pcg_extract(ctx, P, true, n, net, K, eps_r, cfg, opt, C, resid, outer, astats, pstats);
}

int gbem_pcg_extract_cmatrix(gbem_ctx* ctx, const gbem_panels* P, int64_t n, const int32_t* net, int32_t K,
                             double eps_r, const gbem_quad_config* cfg, const gbem_pcg_options* opt, double* C,
                             double* resid, double* outer, gbem_assembly_stats* astats, gbem_pcg_stats* pstats) {
  if (!ctx) return GBEM_EINVAL;
  if (!P || !net || !C || n <= 0) return ctx->fail(GBEM_EINVAL, "null argument or empty panel set");
  if (K < 1 || K > 2048) return ctx->fail(GBEM_EINVAL, "K must be in [1, 2048]");
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  int32_t* d_net = nullptr;
  double* d_out = nullptr;
  GBEM_CUDA(ctx, cudaMallocAsync(&d_net, sizeof(int32_t) * n, ctx->stream));
  GBEM_CUDA(ctx, cudaMallocAsync(&d_out, sizeof(double) * ((size_t)K * K + 2 * K), ctx->stream));
  GBEM_CUDA(ctx, cudaMemcpyAsync(d_net, net, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  int rc = pcg_extract(ctx, P, false, n, d_net, K, eps_r, cfg, opt, d_out, d_out + (size_t)K * K,
                       d_out + (size_t)K * K + K, astats, pstats);
  if (rc == GBEM_OK || ctx->err.find("did not reach") != std::string::npos) {
    GBEM_CUDA(ctx, cudaMemcpyAsync(C, d_out, sizeof(double) * K * K, cudaMemcpyDeviceToHost, ctx->stream));
    if (resid)
      GBEM_CUDA(ctx, cudaMemcpyAsync(resid, d_out + (size_t)K * K, sizeof(double) * K, cudaMemcpyDeviceToHost,
                                     ctx->stream));
    if (outer)
      GBEM_CUDA(ctx, cudaMemcpyAsync(outer, d_out + (size_t)K * K + K, sizeof(double) * K, cudaMemcpyDeviceToHost,
                                     ctx->stream));
  }
  cudaFreeAsync(d_net, ctx->stream);
  cudaFreeAsync(d_out, ctx->stream);
  GBEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return rc;
}

int32_t gbem_ctx_nranks(const gbem_ctx* ctx) { return ctx ? ctx->nranks : 0; }
int32_t gbem_ctx_rank(const gbem_ctx* ctx) { return ctx ? ctx->rank : -1; }

}  // extern "C"

// gbem_capi.cu — the extern "C" boundary declared in include/gbem_gpu.h.
#include <cstring>
#include <new>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "gbem_ctx.cuh"

namespace {

int ensure_matrix(gbem_ctx* ctx, int64_t n, int64_t border = 0) {
  int64_t lda = ((n + border + 7) / 8) * 8;  // 64-byte columns (cp.async alignment)
  if (lda == 0) lda = 8;
  size_t need = (size_t)lda * (size_t)(n + border > 0 ? n + border : 1);
  if (ctx->A_cap < need || !ctx->d_A) {
    if (ctx->d_A) cudaFree(ctx->d_A);
    ctx->d_A = nullptr;
    ctx->A_cap = 0;
    GBEM_CUDA(ctx, cudaMalloc(&ctx->d_A, need * sizeof(double)));
    ctx->A_cap = need;
  }
  ctx->n = n;
  ctx->lda = lda;
  ctx->border = border;
  ctx->factored = false;
  return GBEM_OK;
}

__global__ void k_net_charges(const int32_t* net, int n, const double* X, int nrhs, int K, double scale,
                              double* C, double* outer) {
  // one CTA per rhs; K <= 1024 accumulators in shared memory (deterministic
  // per-thread partials folded in a fixed order)
  extern __shared__ double part[];  // [blockDim.x][K + 1]
  int r = blockIdx.x;
  const int W = K + 1;
  for (int k = 0; k < W; ++k) part[threadIdx.x * W + k] = 0.0;
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    int k = net[p];
    double v = X[(long long)r * n + p];
    part[threadIdx.x * W + (k >= 0 && k < K ? k : K)] += v;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < W; k += blockDim.x) {
    double s = 0.0;
    for (int t = 0; t < (int)blockDim.x; ++t) s += part[t * W + k];
    if (k < K)
      C[(long long)r * K + k] = scale * s;
    else if (outer)
      outer[r] = scale * s;
  }
}

__global__ void k_build_rhs(const int32_t* net, int n, int K, double* B) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)n * K) return;
  int r = (int)(i / n), p = (int)(i % n);
  B[i] = net[p] == r ? 1.0 : 0.0;
}

// Border of the bordered factorisation: row n + q of column c is B(c, q) =
// [net(c) == q]; the K x K corner (columns n..n+K-1, rows n..n+K-1) starts at 0.
__global__ void k_build_border(const int32_t* net, int n, int K, double* A, long long lda) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long cols = (long long)n + K;
  if (i >= cols * K) return;
  const long long c = i / K;
  const int q = (int)(i % K);
  A[c * lda + n + q] = c < n ? (net[c] == q ? 1.0 : 0.0) : 0.0;
}

// C = scale * B^T A^-1 B = -scale * corner (the corner holds -Y^T Y after the
// bordered factorisation; lower triangle, mirrored).  C[r * K + k]: charge of
// net k for unit potential on net r.
__global__ void k_corner_charges(const double* A, long long lda, int n, int K, double scale, double* C) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= K * K) return;
  const int r = i / K, k = i % K;
  const int hi = r > k ? r : k, lo = r > k ? k : r;
  C[i] = -scale * A[(long long)(n + lo) * lda + n + hi];
}

// Nets per extraction: the K border rows ride along every trsm and update of the
// factorisation, so K is bounded only by memory; this cap keeps K*K and the
// border small next to the matrix.
constexpr int32_t kMaxNets = 8192;

int extract_impl(gbem_ctx* ctx, const gbem_panels* P, int64_t n, const int32_t* d_net, int32_t K, double eps_r,
                 const gbem_quad_config* cfg, double* d_C, double* d_resid, gbem_assembly_stats* as,
                 gbem_solve_stats* ss, bool device_panels) {
  if (K < 1 || K > kMaxNets) return ctx->fail(GBEM_EINVAL, "K must be in [1, " + std::to_string(kMaxNets) + "]");
  int rc = gbem_internal_upload_panels(ctx, P, n, device_panels);
  if (rc) return rc;
  rc = ensure_matrix(ctx, n, K);
  if (rc) return rc;
  rc = gbem_internal_assemble(ctx, n, 0, n, cfg, as, true);
  if (rc) return rc;
  size_t cnt = (size_t)n * (size_t)K;
  if (ctx->rhs_cap < cnt) {
    cudaFree(ctx->d_rhs);
    ctx->d_rhs = nullptr;
    ctx->rhs_cap = 0;
    GBEM_CUDA(ctx, cudaMalloc(&ctx->d_rhs, 2 * cnt * sizeof(double)));
    ctx->rhs_cap = cnt;
  }
  double* dB = ctx->d_rhs;
  double* dX = ctx->d_rhs + cnt;
  k_build_rhs<<<(unsigned)((cnt + 255) / 256), 256, 0, ctx->stream>>>(d_net, (int)n, K, dB);
  GBEM_LAUNCH_CHECK(ctx);
  const long long bcnt = ((long long)n + K) * K;
  k_build_border<<<(unsigned)((bcnt + 255) / 256), 256, 0, ctx->stream>>>(d_net, (int)n, K, ctx->d_A, ctx->lda);
  GBEM_LAUNCH_CHECK(ctx);
  // bordered Cholesky: the forward substitution and C = B^T A^-1 B come out of
  // the factorisation; the backward substitution gives X for the residual
  // ||A X - B|| / ||B|| recomputed from the unfactored A (solver.hpp:47)
  rc = gbem_internal_factor(ctx, ss);
  if (rc) return rc;
  if (ss) ss->nrhs = K;
  rc = gbem_internal_solve_factored(ctx, dB, K, dX, d_resid, ss, true);
  if (rc) return rc;
  k_corner_charges<<<(unsigned)((K * K + 255) / 256), 256, 0, ctx->stream>>>(
      ctx->d_A, ctx->lda, (int)n, K, eps_r * 8.854187817e-12 * 1e-6, d_C);
  GBEM_LAUNCH_CHECK(ctx);
  return GBEM_OK;
}

}  // namespace

int gbem_internal_ensure_matrix(gbem_ctx* ctx, int64_t n, int64_t border) { return ensure_matrix(ctx, n, border); }

extern "C" {

int gbem_ctx_create(int device, gbem_ctx** out) {
  if (!out) return GBEM_EINVAL;
  *out = nullptr;
  gbem_ctx* ctx = new (std::nothrow) gbem_ctx();
  if (!ctx) return GBEM_ECUDA;
  *out = ctx;  // the caller can read gbem_last_error even when creation fails
  ctx->device = device;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0 || device < 0 || device >= count) {
    ctx->err = std::string("no CUDA device available: ") + (e != cudaSuccess ? cudaGetErrorString(e) : "device index out of range");
    *out = ctx;  // caller can still read the message
    return GBEM_ECUDA;
  }
  GBEM_CUDA(ctx, cudaSetDevice(device));
  cudaDeviceProp prop;
  GBEM_CUDA(ctx, cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    ctx->err = "this build targets sm_100a (B200); found compute capability " +
               std::to_string(prop.major) + "." + std::to_string(prop.minor);
    *out = ctx;
    return GBEM_ECUDA;
  }
  ctx->num_sms = prop.multiProcessorCount;
  // the warp-cooperative Romberg keeps two tableau rows per lane on the stack
  GBEM_CUDA(ctx, cudaDeviceSetLimit(cudaLimitStackSize, 8192));
  GBEM_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
  ctx->stream = ctx->own_stream;
  // the stream-ordered allocations of a call (work arrays of the host-buffer
  // entry points) stay cached in the pool instead of going back to the driver
  // at every synchronisation
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    cuuint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  for (auto& ev : ctx->ev) GBEM_CUDA(ctx, cudaEventCreate(&ev));
  int rc = gbem_internal_init_tables(ctx);
  *out = ctx;
  return rc;
}

void gbem_ctx_destroy(gbem_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->own_stream) cudaStreamSynchronize(ctx->own_stream);
  if (ctx->stream && ctx->stream != ctx->own_stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->pcg_release) ctx->pcg_release(ctx);
  cudaFree(ctx->d_panels);
  cudaFree(ctx->d_cinfo);
  cudaFree(ctx->d_A);
  cudaFree(ctx->d_diag);
  cudaFree(ctx->d_queue);
  cudaFree(ctx->d_counts);
  cudaFree(ctx->d_offsets);
  cudaFree(ctx->d_cursors);
  cudaFree(ctx->d_stats);
  cudaFree(ctx->d_work);
  cudaFree(ctx->d_info);
  cudaFree(ctx->d_plan);
  cudaFree(ctx->d_flags);
  cudaFree(ctx->d_band_done);
  cudaFree(ctx->d_kp);
  cudaFree(ctx->d_romb);
  cudaFree(ctx->d_queue2);
  cudaFree(ctx->d_plan2);
  cudaFree(ctx->d_offsets2);
  if (ctx->cls_stream) cudaStreamDestroy(ctx->cls_stream);
  for (cudaEvent_t e : ctx->ev_cls)
    if (e) cudaEventDestroy(e);
  cudaFree(ctx->d_romb_cnt);
  cudaFree(ctx->d_rhs);
  cudaFree(ctx->d_linv);
  cudaFree(ctx->d_sw);
  if (ctx->h_stats) cudaFreeHost(ctx->h_stats);
  if (ctx->h_info) cudaFreeHost(ctx->h_info);
  for (auto& ev : ctx->ev)
    if (ev) cudaEventDestroy(ev);
  if (ctx->side_stream) cudaStreamDestroy(ctx->side_stream);
  if (ctx->near_stream) cudaStreamDestroy(ctx->near_stream);
  if (ctx->ev_near_fork) cudaEventDestroy(ctx->ev_near_fork);
  if (ctx->ev_near_join) cudaEventDestroy(ctx->ev_near_join);
  for (int k = 0; k < gbem_ctx::kFarStreams; ++k) {
    if (ctx->far_stream[k]) cudaStreamDestroy(ctx->far_stream[k]);
    if (ctx->ev_far_join[k]) cudaEventDestroy(ctx->ev_far_join[k]);
  }
  if (ctx->ev_panel) cudaEventDestroy(ctx->ev_panel);
  for (auto& e : ctx->ev_bw)
    if (e) cudaEventDestroy(e);
  if (ctx->bw_graph_exec) cudaGraphExecDestroy((cudaGraphExec_t)ctx->bw_graph_exec);
  if (ctx->ev_col) cudaEventDestroy(ctx->ev_col);
  if (ctx->g_side) cudaStreamDestroy(ctx->g_side);
  if (ctx->g_side_lo) cudaStreamDestroy(ctx->g_side_lo);
  if (ctx->g_main) cudaStreamDestroy(ctx->g_main);
  if (ctx->g_main_hi) cudaStreamDestroy(ctx->g_main_hi);
  for (cudaEvent_t e : {ctx->ev_gs, ctx->ev_ge, ctx->ev_gt, ctx->ev_gra, ctx->ev_side_pre, ctx->ev_side_done})
    if (e) cudaEventDestroy(e);
  if (ctx->green_ctx[0] || ctx->green_ctx[1]) {
    PFN_cuGreenCtxDestroy p_destroy = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuGreenCtxDestroy", (void**)&p_destroy, cudaEnableDefault, &q) == cudaSuccess &&
        p_destroy)
      for (void* g : ctx->green_ctx)
        if (g) p_destroy((CUgreenCtx)g);
  }
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

const char* gbem_last_error(const gbem_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int gbem_ctx_set_stream(gbem_ctx* ctx, void* stream) {
  if (!ctx) return GBEM_EINVAL;
  ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  return GBEM_OK;
}

int64_t gbem_ctx_launch_count(const gbem_ctx* ctx) { return ctx ? ctx->launches : 0; }

int gbem_ctx_set_async(gbem_ctx* ctx, int on) {
  if (!ctx) return GBEM_EINVAL;
  ctx->async = on != 0;
  return GBEM_OK;
}

int gbem_ctx_sync(gbem_ctx* ctx) {
  if (!ctx) return GBEM_EINVAL;
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  GBEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  int rc = gbem_internal_check_pending_stats(ctx);
  if (rc) return rc;
  if (ctx->info_pending) {
    ctx->info_pending = false;
    if (*ctx->h_info != 0x7fffffff)
      return ctx->fail(GBEM_ENUMERIC,
                       "matrix not positive definite (pivot at row " + std::to_string(*ctx->h_info) + ")");
  }
  return GBEM_OK;
}

int gbem_u_pair_integrals(gbem_ctx* ctx, const gbem_panels* I, const gbem_panels* J, int64_t npairs,
                          const gbem_quad_config* cfg, double* out, int32_t* converged,
                          gbem_assembly_stats* stats) {
  if (!ctx) return GBEM_EINVAL;
  if (npairs < 0) return ctx->fail(GBEM_EINVAL, "npairs must be >= 0");
  if (npairs == 0) return GBEM_OK;
  if (!I || !J || !out) return ctx->fail(GBEM_EINVAL, "null argument");
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  // concatenate I and J into one panel list: pair k = (k, npairs + k)
  std::vector<uint8_t> ax((size_t)(2 * npairs));
  std::vector<double> lv((size_t)(2 * npairs)), a0(ax.size()), a1(ax.size()), b0(ax.size()), b1(ax.size());
  for (int64_t k = 0; k < npairs; ++k) {
    for (int side = 0; side < 2; ++side) {
      const gbem_panels* S = side ? J : I;
      size_t d = (size_t)(side * npairs + k);
      ax[d] = S->axis[k];
      lv[d] = S->level[k];
      a0[d] = S->a_lo[k];
      a1[d] = S->a_hi[k];
      b0[d] = S->b_lo[k];
      b1[d] = S->b_hi[k];
    }
  }
  gbem_panels all{ax.data(), lv.data(), a0.data(), a1.data(), b0.data(), b1.data()};
  int rc = gbem_internal_upload_panels(ctx, &all, 2 * npairs, false);
  if (rc) return rc;
  double* d_out = nullptr;
  int32_t* d_conv = nullptr;
  GBEM_CUDA(ctx, cudaMallocAsync(&d_out, sizeof(double) * npairs, ctx->stream));
  GBEM_CUDA(ctx, cudaMallocAsync(&d_conv, sizeof(int32_t) * npairs, ctx->stream));
  rc = gbem_internal_pair_list(ctx, npairs, cfg, d_out, d_conv, stats);
  if (rc == GBEM_OK || rc == GBEM_ENUMERIC) {
    GBEM_CUDA(ctx, cudaMemcpyAsync(out, d_out, sizeof(double) * npairs, cudaMemcpyDeviceToHost, ctx->stream));
    if (converged)
      GBEM_CUDA(ctx, cudaMemcpyAsync(converged, d_conv, sizeof(int32_t) * npairs, cudaMemcpyDeviceToHost,
                                     ctx->stream));
  }
  cudaFreeAsync(d_out, ctx->stream);
  cudaFreeAsync(d_conv, ctx->stream);
  GBEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return rc;
}

int gbem_assemble_single(gbem_ctx* ctx, const gbem_panels* P, int64_t n, const gbem_quad_config* cfg,
                         double* A_host, int64_t lda, gbem_assembly_stats* stats) {
  if (!ctx) return GBEM_EINVAL;
  if (A_host && lda < n) return ctx->fail(GBEM_EINVAL, "lda < n");
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  int rc = gbem_internal_upload_panels(ctx, P, n, false);
  if (rc) return rc;
  rc = ensure_matrix(ctx, n);
  if (rc) return rc;
  rc = gbem_internal_assemble(ctx, n, 0, n, cfg, stats, true);
  if (rc) return rc;
  if (A_host) return gbem_matrix_download(ctx, A_host, lda);
  GBEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return GBEM_OK;
}

int gbem_assemble_single_dev(gbem_ctx* ctx, const gbem_panels* P, int64_t n, const gbem_quad_config* cfg,
                             gbem_assembly_stats* stats) {
  if (!ctx) return GBEM_EINVAL;
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  int rc = gbem_internal_upload_panels(ctx, P, n, true);
  if (rc) return rc;
  rc = ensure_matrix(ctx, n);
  if (rc) return rc;
  return gbem_internal_assemble(ctx, n, 0, n, cfg, stats, true);
}

int gbem_assemble_rows_dev(gbem_ctx* ctx, const gbem_panels* P, int64_t n, int64_t row_begin, int64_t row_end,
                           const gbem_quad_config* cfg, double* out, int64_t ld_out, gbem_assembly_stats* stats) {
  if (!ctx) return GBEM_EINVAL;
  if (row_begin < 0 || row_end > n || row_begin > row_end)
    return ctx->fail(GBEM_EINVAL, "row range out of bounds");
  if (!out || ld_out < n) return ctx->fail(GBEM_EINVAL, "row block buffer missing or ld_out < n");
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  int rc = gbem_internal_upload_panels(ctx, P, n, true);
  if (rc) return rc;
  if (row_end == row_begin) return GBEM_OK;
  return gbem_internal_assemble(ctx, n, row_begin, row_end, cfg, stats, false, out, ld_out);
}

int gbem_assemble_rows_full_dev(gbem_ctx* ctx, const gbem_panels* P, int64_t n, int64_t row_begin,
                                int64_t row_end, const gbem_quad_config* cfg, double* out, int64_t ld_out,
                                gbem_assembly_stats* stats) {
  if (!ctx) return GBEM_EINVAL;
  if (row_begin < 0 || row_end > n || row_begin > row_end)
    return ctx->fail(GBEM_EINVAL, "row range out of bounds");
  if (!out || ld_out < n) return ctx->fail(GBEM_EINVAL, "row block buffer missing or ld_out < n");
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  int rc = gbem_internal_upload_panels(ctx, P, n, true);
  if (rc) return rc;
  if (row_end == row_begin) return GBEM_OK;
  return gbem_internal_assemble(ctx, n, row_begin, row_end, cfg, stats, false, out, ld_out, true);
}

int gbem_rowblock_matvec_dev(gbem_ctx* ctx, const double* Ablk, int64_t ld, int64_t rows, int64_t n,
                             const double* P, int64_t ldp, int64_t K, double* Q, int64_t ldq) {
  if (!ctx) return GBEM_EINVAL;
  if (!Ablk || !P || !Q || ld < n || rows < 0 || K < 0 || ldp < K || ldq < K)
    return ctx->fail(GBEM_EINVAL, "bad row-block matvec arguments");
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  return gbem_internal_rowblock_matvec(ctx, Ablk, ld, rows, n, P, ldp, K, Q, ldq);
}

int gbem_spd_factor_dev(gbem_ctx* ctx, const double* M, int64_t m, int64_t ldm, gbem_solve_stats* stats) {
  if (!ctx) return GBEM_EINVAL;
  if (m < 0 || (m > 0 && (!M || ldm < m))) return ctx->fail(GBEM_EINVAL, "bad matrix dimensions");
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  int rc = ensure_matrix(ctx, m);
  if (rc) return rc;
  if (m > 0)
    GBEM_CUDA(ctx, cudaMemcpy2DAsync(ctx->d_A, sizeof(double) * ctx->lda, M, sizeof(double) * ldm, sizeof(double) * m,
                                     m, cudaMemcpyDeviceToDevice, ctx->stream));
  return gbem_internal_factor(ctx, stats);
}

int gbem_matrix_apply_dev(gbem_ctx* ctx, const double* X, int64_t nrhs, double* Y) {
  if (!ctx) return GBEM_EINVAL;
  if (!X || !Y) return ctx->fail(GBEM_EINVAL, "null argument");
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  int rc = gbem_internal_apply(ctx, X, nrhs, Y);
  if (rc) return rc;
  if (!ctx->async) GBEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return GBEM_OK;
}

int gbem_spd_solve_factored_dev(gbem_ctx* ctx, const double* B, int64_t nrhs, double* X, double* resid,
                                gbem_solve_stats* stats) {
  if (!ctx) return GBEM_EINVAL;
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  return gbem_internal_solve_factored(ctx, B, nrhs, X, resid, stats);
}

int gbem_assemble_collocation(gbem_ctx* ctx, const gbem_block_panels* P, int64_t n, const gbem_region* regions,
                              int32_t nregions, int32_t main_net, double* A_host, int64_t lda, double* b_host,
                              int64_t* m_out) {
  if (!ctx) return GBEM_EINVAL;
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  int64_t m = 0;
  int rc = gbem_internal_assemble_collocation(ctx, P, n, regions, nregions, main_net, &m);
  if (rc) return rc;
  ctx->block_m = m;
  if (m_out) *m_out = m;
  if (A_host) {  // row-major copy of the column-major device matrix
    if (lda < m) return ctx->fail(GBEM_EINVAL, "lda < m");
    std::vector<double> t((size_t)ctx->lda * m);
    GBEM_CUDA(ctx, cudaMemcpy(t.data(), ctx->d_A, sizeof(double) * t.size(), cudaMemcpyDeviceToHost));
    for (int64_t r = 0; r < m; ++r)
      for (int64_t c = 0; c < m; ++c) A_host[r * lda + c] = t[(size_t)c * ctx->lda + r];
  }
  if (b_host) GBEM_CUDA(ctx, cudaMemcpy(b_host, ctx->d_rhs, sizeof(double) * m, cudaMemcpyDeviceToHost));
  return GBEM_OK;
}

int gbem_assemble_multi(gbem_ctx* ctx, const gbem_block_panels* P, int64_t n, const gbem_region* regions,
                        int32_t nregions, int32_t main_net, const gbem_quad_config* cfg, double* A_host, int64_t lda,
                        double* b_host, int64_t* m_out, int32_t* all_converged) {
  if (!ctx) return GBEM_EINVAL;
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  int64_t m = 0, nonconv = 0;
  int rc = gbem_internal_assemble_block(ctx, P, n, regions, nregions, main_net, true, cfg, &m, &nonconv);
  if (rc) return rc;
  ctx->block_m = m;
  if (m_out) *m_out = m;
  if (all_converged) *all_converged = nonconv == 0 ? 1 : 0;
  if (A_host) {  // row-major copy of the column-major device matrix
    if (lda < m) return ctx->fail(GBEM_EINVAL, "lda < m");
    std::vector<double> t((size_t)ctx->lda * m);
    GBEM_CUDA(ctx, cudaMemcpy(t.data(), ctx->d_A, sizeof(double) * t.size(), cudaMemcpyDeviceToHost));
    for (int64_t r = 0; r < m; ++r)
      for (int64_t c = 0; c < m; ++c) A_host[r * lda + c] = t[(size_t)c * ctx->lda + r];
  }
  if (b_host) GBEM_CUDA(ctx, cudaMemcpy(b_host, ctx->d_rhs, sizeof(double) * m, cudaMemcpyDeviceToHost));
  return GBEM_OK;
}

int gbem_oracle_pair_integrals(gbem_ctx* ctx, const gbem_panels* I, const gbem_panels* J, const int32_t* nsign,
                               int64_t npairs, int32_t double_layer, int32_t depth, double* out) {
  if (!ctx) return GBEM_EINVAL;
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  return gbem_internal_oracle_pairs(ctx, I, J, nsign, npairs, double_layer, depth, out);
}

int gbem_selftest(gbem_ctx* ctx, int32_t pairs, uint64_t seed, const gbem_quad_config* cfg,
                  gbem_selftest_case* cases, int32_t* ncases) {
  if (!ctx) return GBEM_EINVAL;
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  return gbem_internal_selftest(ctx, pairs, seed, cfg, cases, ncases);
}

int gbem_matrix_upload_general(gbem_ctx* ctx, const double* A_host, int64_t n, int64_t lda) {
  if (!ctx || (!A_host && n > 0)) return GBEM_EINVAL;
  if (n < 0 || lda < n) return ctx->fail(GBEM_EINVAL, "bad matrix dimensions");
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  int rc = ensure_matrix(ctx, n);
  if (rc) return rc;
  if (n == 0) return GBEM_OK;
  std::vector<double> t((size_t)n * ctx->lda, 0.0);  // column-major image of the row-major input
  for (int64_t r = 0; r < n; ++r)
    for (int64_t c = 0; c < n; ++c) t[(size_t)c * ctx->lda + r] = A_host[r * lda + c];
  GBEM_CUDA(ctx, cudaMemcpy(ctx->d_A, t.data(), sizeof(double) * t.size(), cudaMemcpyHostToDevice));
  ctx->block_m = -1;
  return GBEM_OK;
}

int gbem_lu_solve(gbem_ctx* ctx, const double* b_host, double* x_host, double* resid, gbem_solve_stats* stats) {
  if (!ctx) return GBEM_EINVAL;
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  const int64_t m = ctx->n;
  if (ctx->factored) return ctx->fail(GBEM_EINVAL, "matrix already factored; re-assemble or re-upload");
  if (!b_host && ctx->block_m != m) return ctx->fail(GBEM_EINVAL, "no assembled right-hand side; pass b");
  if (m > 0 && !x_host) return ctx->fail(GBEM_EINVAL, "null solution buffer");
  if (ctx->rhs_cap < (size_t)m || !ctx->d_rhs) {
    cudaFree(ctx->d_rhs);
    ctx->d_rhs = nullptr;
    ctx->rhs_cap = 0;
    GBEM_CUDA(ctx, cudaMalloc(&ctx->d_rhs, 2 * (size_t)(m > 0 ? m : 1) * sizeof(double)));
    ctx->rhs_cap = m;
  }
  double* d_b = ctx->d_rhs;
  double* d_x = ctx->d_rhs + m;
  if (b_host) GBEM_CUDA(ctx, cudaMemcpy(d_b, b_host, sizeof(double) * m, cudaMemcpyHostToDevice));
  double* d_r = nullptr;
  GBEM_CUDA(ctx, cudaMalloc(&d_r, sizeof(double)));
  int rc = gbem_internal_lu_solve(ctx, d_b, d_x, d_r, stats);
  ctx->block_m = -1;
  if (rc == GBEM_OK) {
    if (m > 0) GBEM_CUDA(ctx, cudaMemcpy(x_host, d_x, sizeof(double) * m, cudaMemcpyDeviceToHost));
    if (resid) GBEM_CUDA(ctx, cudaMemcpy(resid, d_r, sizeof(double), cudaMemcpyDeviceToHost));
  }
  cudaFree(d_r);
  return rc;
}

int gbem_matrix_download(gbem_ctx* ctx, double* A_host, int64_t lda) {
  if (!ctx || !A_host) return GBEM_EINVAL;
  if (lda < ctx->n) return ctx->fail(GBEM_EINVAL, "lda < n");
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  // column-major device == row-major host for the symmetric matrix; a factored
  // matrix comes back as its column-major lower factor transposed.
  GBEM_CUDA(ctx, cudaMemcpy2DAsync(A_host, sizeof(double) * lda, ctx->d_A, sizeof(double) * ctx->lda,
                                   sizeof(double) * ctx->n, ctx->n, cudaMemcpyDeviceToHost, ctx->stream));
  GBEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return GBEM_OK;
}

int gbem_matrix_upload(gbem_ctx* ctx, const double* A_host, int64_t n, int64_t lda) {
  if (!ctx || (!A_host && n > 0)) return GBEM_EINVAL;
  if (n < 0 || lda < n) return ctx->fail(GBEM_EINVAL, "bad matrix dimensions");
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  int rc = ensure_matrix(ctx, n);
  if (rc) return rc;
  if (n == 0) return GBEM_OK;
  // row-major host -> column-major device of the transpose (== A when symmetric)
  GBEM_CUDA(ctx, cudaMemcpy2DAsync(ctx->d_A, sizeof(double) * ctx->lda, A_host, sizeof(double) * lda,
                                   sizeof(double) * n, n, cudaMemcpyHostToDevice, ctx->stream));
  GBEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return GBEM_OK;
}

int gbem_matrix_device(gbem_ctx* ctx, double** A_dev, int64_t* n, int64_t* lda) {
  if (!ctx) return GBEM_EINVAL;
  if (A_dev) *A_dev = ctx->d_A;
  if (n) *n = ctx->n;
  if (lda) *lda = ctx->lda;
  return GBEM_OK;
}

int gbem_spd_solve(gbem_ctx* ctx, const double* B, int64_t nrhs, double* X, double* resid,
                   gbem_solve_stats* stats) {
  if (!ctx) return GBEM_EINVAL;
  if (nrhs < 0) return ctx->fail(GBEM_EINVAL, "cholesky_solve: dimension mismatch");
  if (nrhs > 0 && (!B || !X)) return ctx->fail(GBEM_EINVAL, "null argument");
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  const int64_t n = ctx->n;
  size_t cnt = (size_t)n * (size_t)nrhs;
  double *dB = nullptr, *dX = nullptr, *dR = nullptr;
  if (cnt) {
    GBEM_CUDA(ctx, cudaMalloc(&dB, cnt * sizeof(double)));
    GBEM_CUDA(ctx, cudaMalloc(&dX, cnt * sizeof(double)));
    GBEM_CUDA(ctx, cudaMalloc(&dR, (size_t)nrhs * sizeof(double)));
    GBEM_CUDA(ctx, cudaMemcpyAsync(dB, B, cnt * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  }
  int rc = gbem_internal_solve(ctx, dB, nrhs, dX, dR, stats);
  if (rc == GBEM_OK && cnt) {
    GBEM_CUDA(ctx, cudaMemcpyAsync(X, dX, cnt * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    if (resid)
      GBEM_CUDA(ctx, cudaMemcpyAsync(resid, dR, (size_t)nrhs * sizeof(double), cudaMemcpyDeviceToHost,
                                     ctx->stream));
  }
  cudaStreamSynchronize(ctx->stream);
  cudaFree(dB);
  cudaFree(dX);
  cudaFree(dR);
  return rc;
}

int gbem_spd_solve_dev(gbem_ctx* ctx, const double* B, int64_t nrhs, double* X, double* resid,
                       gbem_solve_stats* stats) {
  if (!ctx) return GBEM_EINVAL;
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  return gbem_internal_solve(ctx, B, nrhs, X, resid, stats);
}

namespace {
__global__ void k_fill_shared(double value, int words) {
  extern __shared__ double fill_sm[];
  for (int i = threadIdx.x; i < words; i += blockDim.x) fill_sm[i] = value;
  __syncthreads();
  // keep the stores: an impossible condition on the data read back
  if (fill_sm[(threadIdx.x * 7) % words] == 1.2345e-300 && value != 1.2345e-300) fill_sm[0] = 0.0;
}
}  // namespace

int gbem_debug_fill_shared(gbem_ctx* ctx, double value) {
  if (!ctx) return GBEM_EINVAL;
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  int maxsm = 0;
  GBEM_CUDA(ctx, cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  GBEM_CUDA(ctx, cudaFuncSetAttribute(k_fill_shared, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
  k_fill_shared<<<ctx->num_sms * 2, 1024, maxsm, ctx->stream>>>(value, maxsm / 8);
  GBEM_LAUNCH_CHECK(ctx);
  GBEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return GBEM_OK;
}

int gbem_net_charges_dev(gbem_ctx* ctx, const int32_t* net, int64_t n, const double* X, int64_t nrhs,
                         int32_t K, double scale, double* C, double* outer) {
  if (!ctx) return GBEM_EINVAL;
  if (K < 1 || K > 512 || nrhs < 0) return ctx->fail(GBEM_EINVAL, "net count must be in [1, 512]");
  if (nrhs == 0 || n == 0) return GBEM_OK;
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  int threads = 64;
  size_t smem = sizeof(double) * (size_t)threads * (size_t)(K + 1);
  if (smem > 200 * 1024) return ctx->fail(GBEM_EINVAL, "too many nets for the charge reduction");
  if (smem > 48 * 1024)
    GBEM_CUDA(ctx, cudaFuncSetAttribute(k_net_charges, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_net_charges<<<(unsigned)nrhs, threads, smem, ctx->stream>>>(net, (int)n, X, (int)nrhs, K, scale, C, outer);
  GBEM_LAUNCH_CHECK(ctx);
  return GBEM_OK;
}

int gbem_extract_cmatrix(gbem_ctx* ctx, const gbem_panels* P, int64_t n, const int32_t* net_of_panel, int32_t K,
                         double eps_r, const gbem_quad_config* cfg, double* C, double* resid,
                         gbem_assembly_stats* as, gbem_solve_stats* ss) {
  if (!ctx) return GBEM_EINVAL;
  if (!P || !net_of_panel || !C || n <= 0) return ctx->fail(GBEM_EINVAL, "null argument or empty panel set");
  if (K < 1 || K > kMaxNets) return ctx->fail(GBEM_EINVAL, "K must be in [1, " + std::to_string(kMaxNets) + "]");
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  if (ctx->nranks > 1) {
    // ranks attached (gbem_ctx_init_nccl / gbem_ctx_set_collectives): the matrix is
    // sharded by row blocks and solved by block-Jacobi PCG (gbem_pcg.cu), Jacobi
    // blocks of ~12k rows (the 8-rank config-4 shape)
    const int64_t rows = (n + ctx->nranks - 1) / ctx->nranks;
    gbem_pcg_options po{1e-10, 5000, (int32_t)std::max<int64_t>(1, (rows + 12031) / 12032)};
    if (ss) *ss = gbem_solve_stats{};
    return gbem_pcg_extract_cmatrix(ctx, P, n, net_of_panel, K, eps_r, cfg, &po, C, resid, nullptr, as, nullptr);
  }
  int32_t* d_net = nullptr;
  double *d_C = nullptr, *d_res = nullptr;
  GBEM_CUDA(ctx, cudaMallocAsync(&d_net, sizeof(int32_t) * n, ctx->stream));
  GBEM_CUDA(ctx, cudaMallocAsync(&d_C, sizeof(double) * ((size_t)K * K + K), ctx->stream));
  d_res = d_C + (size_t)K * K;
  GBEM_CUDA(ctx, cudaMemcpyAsync(d_net, net_of_panel, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  int rc = extract_impl(ctx, P, n, d_net, K, eps_r, cfg, d_C, d_res, as, ss, false);
  if (rc == GBEM_OK) {
    GBEM_CUDA(ctx, cudaMemcpyAsync(C, d_C, sizeof(double) * K * K, cudaMemcpyDeviceToHost, ctx->stream));
    if (resid) GBEM_CUDA(ctx, cudaMemcpyAsync(resid, d_res, sizeof(double) * K, cudaMemcpyDeviceToHost, ctx->stream));
  }
  cudaFreeAsync(d_net, ctx->stream);
  cudaFreeAsync(d_C, ctx->stream);
  GBEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return rc;
}

int gbem_extract_cmatrix_dev(gbem_ctx* ctx, const gbem_panels* P, int64_t n, const int32_t* net_of_panel,
                             int32_t K, double eps_r, const gbem_quad_config* cfg, double* C, double* resid,
                             gbem_assembly_stats* as, gbem_solve_stats* ss) {
  if (!ctx) return GBEM_EINVAL;
  if (!P || !net_of_panel || !C || n <= 0) return ctx->fail(GBEM_EINVAL, "null argument or empty panel set");
  GBEM_CUDA(ctx, cudaSetDevice(ctx->device));
  if (ctx->nranks > 1) {  // sharded solve, as in gbem_extract_cmatrix
    const int64_t rows = (n + ctx->nranks - 1) / ctx->nranks;
    gbem_pcg_options po{1e-10, 5000, (int32_t)std::max<int64_t>(1, (rows + 12031) / 12032)};
    if (ss) *ss = gbem_solve_stats{};
    return gbem_pcg_extract_cmatrix_dev(ctx, P, n, net_of_panel, K, eps_r, cfg, &po, C, resid, nullptr, as, nullptr);
  }
  return extract_impl(ctx, P, n, net_of_panel, K, eps_r, cfg, C, resid, as, ss, true);
}

}  // extern "C"

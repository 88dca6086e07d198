// gbem_ctx.cuh — internal context shared by the assembly, solver and C-ABI units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/gbem_gpu.h"
#include "gbem_common.cuh"

struct gbem_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;      // active stream
  cudaStream_t own_stream = nullptr;  // created by the context
  std::string err;
  int64_t launches = 0;
  int num_sms = 148;

  // panels (device, 48-byte records)
  gbem_gpu::DPanel* d_panels = nullptr;
  int64_t panel_cap = 0;
  void* d_cinfo = nullptr;  // per-panel classification records (gbem_assembly.cu CPanel)
  int64_t cinfo_cap = 0;

  // matrix: column-major n x n with leading dimension lda (symmetric after
  // assembly; lower triangle overwritten by the Cholesky factor)
  double* d_A = nullptr;
  int64_t n = 0, lda = 0;
  // bordered factorisation (K-RHS extraction): `border` rows below the matrix
  // hold B^T (the net incidence) and a border x border corner block starts at
  // zero; the Cholesky then carries them along, leaving Y^T = (L^-1 B)^T in the
  // border rows and -Y^T Y = -B^T A^-1 B in the corner (the forward
  // substitution and the charge reduction fused into the factorisation)
  int64_t border = 0;
  size_t A_cap = 0;  // elements
  double* d_diag = nullptr;  // original diagonal (kept for residuals after factoring)
  int64_t diag_cap = 0;
  bool factored = false;
  int64_t block_m = -1;  // size of the assembled block system whose b sits in d_rhs (-1: none)
  // stream-ordered mode (gbem_ctx_set_async): the factorisation's pivot check is
  // read back at gbem_ctx_sync instead of blocking inside the call
  bool async = false;
  bool info_pending = false;
  bool stats_pending = false;

  // assembly work buffers
  uint64_t* d_queue = nullptr;
  int64_t queue_cap = 0;
  uint32_t* d_plan = nullptr;  // far-field plan per queue entry (gbem_assembly.cu, far_plan_code)
  int64_t plan_cap = 0;
  uint64_t* d_kp = nullptr;  // (key, plan) per pair in tile order between the two classification passes
  int64_t kp_cap = 0;
  // second queue / plan / offsets set: chunk t + 1 is classified (on cls_stream) while chunk t is evaluated
  uint64_t* d_queue2 = nullptr;
  int64_t queue2_cap = 0;
  uint32_t* d_plan2 = nullptr;
  int64_t plan2_cap = 0;
  uint32_t* d_offsets2 = nullptr;
  cudaStream_t cls_stream = nullptr;
  cudaEvent_t ev_cls[5] = {};  // fork, classified[2], evaluated[2]
  // near-contact (Romberg-route) pairs collected over the chunks of one assembly and evaluated
  // together at its end: entries, then {count, taken from the current chunk}
  uint64_t* d_romb = nullptr;
  uint32_t* d_romb_cnt = nullptr;
  uint32_t* d_counts = nullptr;   // per key
  uint32_t* d_offsets = nullptr;  // exclusive scan of counts (kNumKeys + 1)
  uint32_t* d_cursors = nullptr;
  unsigned long long* d_stats = nullptr;  // device counters (see gbem_assembly.cu)
  unsigned long long* h_stats = nullptr;  // pinned mirror

  // solver work buffers
  double* d_work = nullptr;
  size_t work_cap = 0;  // elements
  int* d_info = nullptr;
  int* h_info = nullptr;  // pinned
  double* d_sw = nullptr;  // blocked multi-RHS solve: W, Y, X (3 n R)
  size_t sw_cap = 0;
  double* d_linv = nullptr;  // inverses of the 128 x 128 diagonal blocks of the factor
  size_t linv_cap = 0;
  int* d_flags = nullptr;  // per-block ready flags of the dataflow backward substitution
  int flow_epoch = 0;
  unsigned* d_band_done = nullptr;  // finished look-ahead band tiles of the factor (counter)
  double* d_rhs = nullptr;  // B and X of the K-RHS extraction (2 * rhs_cap)
  size_t rhs_cap = 0;

  cudaEvent_t ev[8] = {};
  cudaStream_t side_stream = nullptr;  // high-priority look-ahead stream of the factorisation
  cudaEvent_t ev_panel = nullptr, ev_col = nullptr;
  // near-field kernels of an assembly chunk run beside its far-field kernels (gbem_assembly.cu run_eval)
  cudaStream_t near_stream = nullptr;
  cudaEvent_t ev_near_fork = nullptr, ev_near_join = nullptr;
  // the far-field kernels of a chunk are dealt over the caller's stream and these (their tails overlap)
  static constexpr int kFarStreams = 3;
  cudaStream_t far_stream[kFarStreams] = {};
  cudaEvent_t ev_far_join[kFarStreams] = {};
  cudaEvent_t ev_bw[5] = {};  // look-ahead backward substitution: start, step done, bulk done x 3
  // its captured sweep (cudaGraphExec_t), valid for one (matrix, factor, work, output, shape) tuple
  struct BwdGraphKey {
    const void *A = nullptr, *linv = nullptr, *work = nullptr, *out = nullptr;
    int64_t lda = 0;
    int n = 0, R = 0;
    bool operator==(const BwdGraphKey& o) const {
      return A == o.A && linv == o.linv && work == o.work && out == o.out && lda == o.lda && n == o.n && R == o.R;
    }
  };
  void* bw_graph_exec = nullptr;
  BwdGraphKey bw_graph_key;
  int64_t bw_graph_launches = 0;
  // SM-partitioned factorisation (green contexts): the diagonal-block factor
  // runs on a reserved SM pair (g_side) while the trailing updates run on the
  // other SMs (g_main); otherwise the update CTAs fill every SM and the
  // full-SM factor kernel waits for an SM to drain.  green_state: 0 untried,
  // 1 available, -1 unavailable (fall back to side_stream in the primary context).
  int green_state = 0;
  int green_side_sms = 0;
  cudaStream_t g_main = nullptr, g_main_hi = nullptr, g_side = nullptr;
  cudaStream_t g_side_lo = nullptr;  // low-priority stream of the side partition: a share of the large updates
  cudaEvent_t ev_side_pre = nullptr, ev_side_done = nullptr;
  cudaEvent_t ev_gs = nullptr, ev_ge = nullptr, ev_gt = nullptr, ev_gra = nullptr;
  void* green_ctx[2] = {nullptr, nullptr};  // CUgreenCtx (side, main)

  // row-block sharded solve (gbem_pcg.cu): ranks and collectives
  int32_t nranks = 1, rank = 0;
  void* nccl_comm = nullptr;           // ncclComm_t owned by the context (gbem_ctx_init_nccl)
  gbem_collectives coll{};             // host-provided collectives (gbem_ctx_set_collectives)
  bool has_coll = false;
  void* pcg_ws = nullptr;              // sharded-solve workspace (gbem_pcg.cu)
  void (*pcg_release)(gbem_ctx*) = nullptr;  // frees pcg_ws and the communicator

  // kernels whose dynamic shared-memory limit has been raised on this
  // context's device (cudaFuncSetAttribute is per device; one bit per site)
  uint64_t attr_set = 0;
  enum : uint64_t { kAttrGemmSolve = 1u, kAttrFactor = 2u, kAttrGemmLU = 4u, kAttrPcgGemm = 8u, kAttrSymm = 16u, kAttrBwdStep = 32u };

  int fail(int code, const std::string& msg) {
    err = msg;
    return code;
  }
};

// Wrap a CUDA runtime call inside a C-ABI entry point.
#define GBEM_CUDA(ctx, call)                                                              \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return (ctx)->fail(GBEM_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define GBEM_LAUNCH_CHECK(ctx)                                                            \
  do {                                                                                    \
    (ctx)->launches++;                                                                    \
    cudaError_t e_ = cudaGetLastError();                                                  \
    if (e_ != cudaSuccess)                                                                \
      return (ctx)->fail(GBEM_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

// Internal entry points implemented across the units.
int gbem_internal_ensure_matrix(gbem_ctx* ctx, int64_t n, int64_t border = 0);
int gbem_internal_assemble_collocation(gbem_ctx* ctx, const gbem_block_panels* P, int64_t n,
                                       const gbem_region* regions, int32_t nreg, int32_t main_net, int64_t* m_out);
int gbem_internal_assemble_block(gbem_ctx* ctx, const gbem_block_panels* P, int64_t n, const gbem_region* regions,
                                 int32_t nreg, int32_t main_net, bool galerkin, const gbem_quad_config* cfg,
                                 int64_t* m_out, int64_t* nonconv_out);
int gbem_internal_lu_solve(gbem_ctx* ctx, double* d_b, double* d_x, double* d_resid, gbem_solve_stats* stats);
int gbem_internal_upload_panels(gbem_ctx* ctx, const gbem_panels* P, int64_t n, bool device_ptrs);
int gbem_internal_check_pending_stats(gbem_ctx* ctx);
int gbem_internal_assemble(gbem_ctx* ctx, int64_t n, int64_t row_begin, int64_t row_end,
                           const gbem_quad_config* cfg, gbem_assembly_stats* stats, bool symmetrize,
                           double* out = nullptr, int64_t ld_out = 0, bool full_rows = false,
                           bool out_col_major = false);
int gbem_internal_rowblock_matvec(gbem_ctx* ctx, const double* Ab, int64_t ld, int64_t rows, int64_t n,
                                  const double* P, int64_t ldp, int64_t K, double* Q, int64_t ldq);
int gbem_internal_pair_list(gbem_ctx* ctx, int64_t npairs, const gbem_quad_config* cfg,
                            double* d_out, int32_t* d_conv, gbem_assembly_stats* stats);
int gbem_internal_init_tables(gbem_ctx* ctx);
int gbem_internal_oracle_pairs(gbem_ctx* ctx, const gbem_panels* I, const gbem_panels* J, const int32_t* nsign,
                               int64_t npairs, int32_t dbl, int32_t depth, double* out);
int gbem_internal_selftest(gbem_ctx* ctx, int32_t pairs, uint64_t seed, const gbem_quad_config* cfg,
                           gbem_selftest_case* cases, int32_t* ncases);
int gbem_internal_apply(gbem_ctx* ctx, const double* d_X, int64_t nrhs, double* d_Y);
int gbem_internal_solve(gbem_ctx* ctx, const double* d_B, int64_t nrhs, double* d_X,
                        double* d_resid, gbem_solve_stats* stats);
int gbem_internal_factor(gbem_ctx* ctx, gbem_solve_stats* stats);
int gbem_internal_solve_factored(gbem_ctx* ctx, const double* d_B, int64_t nrhs, double* d_X, double* d_resid,
                                 gbem_solve_stats* stats, bool y_from_border = false);

/* gbem_gpu.h — C-ABI boundary of the B200-native GBEM hot path.
 *
 * Replaces, for the single-dielectric Galerkin path of the reference
 * (arxiv 2203.11733 code, /root/reference/proj):
 *   - u_pair_integral            proj/include/gbem/kernels.hpp:270   -> gbem_u_pair_integrals
 *   - assemble_single            proj/include/gbem/assembly.hpp:82   -> gbem_assemble_single(_dev)
 *   - cholesky_solve             proj/include/gbem/solver.hpp:24     -> gbem_spd_solve(_dev)
 *   - net_charges (Q = eps_r*eps0*X*1e-6 summed per net)
 *                                proj/include/gbem/extraction.hpp:55 -> gbem_net_charges_dev
 *   - dump_system_matrix layout  proj/include/gbem/extraction.hpp:83 -> gbem_matrix_download
 *
 * Plain C types only.  Every function returns a status code:
 *   GBEM_OK 0, GBEM_EINVAL 1 (ValidationError, exit 1), GBEM_ENUMERIC 2
 *   (NumericalError, exit 2: non-finite quadrature sample, non-SPD pivot),
 *   GBEM_ECUDA 3 (CUDA runtime failure / no device).
 * The message for the last failure of a context is gbem_last_error(ctx).
 * Errors mirror proj/include/gbem/errors.hpp:10-20.
 *
 * Threading: one context per host thread; calls are stream-ordered on the
 * context's stream and the host-buffer variants block until their results are
 * in host memory.  No global state besides the per-device constant tables.
 */
#ifndef GBEM_GPU_H
#define GBEM_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GBEM_OK 0
#define GBEM_EINVAL 1
#define GBEM_ENUMERIC 2
#define GBEM_ECUDA 3

typedef struct gbem_ctx gbem_ctx;

/* Panel list in structure-of-arrays form (Rect, geometry.hpp:52-76): panel k lies
 * in the plane x[axis[k]] == level[k], spanning [a_lo,a_hi] x [b_lo,b_hi] along
 * the in-plane axes in axis-index order.  All arrays have n entries.  Host or
 * device pointers depending on the entry point. */
typedef struct {
  const uint8_t* axis;
  const double* level;
  const double* a_lo;
  const double* a_hi;
  const double* b_lo;
  const double* b_hi;
} gbem_panels;

/* QuadratureConfig (quadrature.hpp:12-15) for the near-field Romberg path plus
 * the far-field split.  Zero-initialised fields take the defaults:
 * rel_tol 1e-8, max_levels 16, near_ratio 1.0 (>= 1; pairs with gap < near_ratio *
 * max diameter use the reference's semi-analytic forms; the rest use the
 * anisotropic tensor-Gauss rule), far_tol 1e-12 (target relative error of the
 * far-field rule). */
typedef struct {
  double rel_tol;
  int32_t max_levels;
  double near_ratio;
  double far_tol;
} gbem_quad_config;

typedef struct {
  int64_t pairs_total;       /* unique pairs evaluated, n(n+1)/2 for a matrix */
  int64_t pairs_coplanar;    /* closed-form coplanar (incl. self) */
  int64_t pairs_parallel;    /* near offset-parallel, Romberg */
  int64_t pairs_orthogonal;  /* near orthogonal, Romberg */
  int64_t pairs_far;         /* anisotropic tensor Gauss */
  int64_t not_converged;     /* Romberg hit max_levels (QuadStats::converged) */
  int64_t nonfinite;         /* non-finite integrand samples (NumericalError) */
  int64_t near_evals;        /* Romberg integrand samples */
  int64_t far_evals;         /* Gauss kernel evaluations */
  double far_flops;          /* algorithmic FP64 flops of the far kernel */
  double ms_classify, ms_far, ms_near, ms_total; /* device time per phase */
  /* near-field routes (included in pairs_parallel + pairs_orthogonal):
   * gap < 1e-3 max diameter -> the reference's adaptive Romberg (warp per pair);
   * band b -> graded Gauss-Legendre, gap/diam in [0.1, 1) or touching (b = 0),
   * [0.02, 0.1) (1), [0.005, 0.02) (2), [1e-3, 0.005) (3) */
  int64_t pairs_near_romberg;
  int64_t pairs_near_band[4];
} gbem_assembly_stats;

typedef struct {
  int64_t n;
  int64_t nrhs;
  int64_t bad_pivot;         /* first non-positive pivot row, -1 if none */
  double max_residual;       /* max over rhs of ||A x - b|| / ||b|| (solver.hpp:17-21) */
  double ms_factor, ms_solve, ms_residual;
} gbem_solve_stats;

/* Block (mixed-unknown) system panels (Panel, partition.hpp:34-46), class-
 * contiguous [conductor, dirichlet outer, neumann outer, interface]; host arrays. */
typedef struct {
  gbem_panels geom;
  const int8_t* nsign;   /* Rect::normalSign, +1 / -1 */
  const int32_t* kind;   /* 0 conductor, 1 dirichlet outer, 2 neumann outer, 3 interface */
  const int32_t* net;    /* net id (conductor panels) */
  const int32_t* reg_a;  /* regionA */
  const int32_t* reg_b;  /* regionB (interface panels) */
} gbem_block_panels;

/* DielectricRegion id and relative permittivity. */
typedef struct {
  int32_t id;
  double eps;
} gbem_region;

/* Context on CUDA device `device` (one process per GPU; ranks pick their own). */
int gbem_ctx_create(int device, gbem_ctx** out);
void gbem_ctx_destroy(gbem_ctx* ctx);
const char* gbem_last_error(const gbem_ctx* ctx);
/* Run subsequent work on an existing cudaStream_t (NULL: the context's own
 * non-blocking stream; pass cudaStreamLegacy, (void*)1, for the legacy default
 * stream, which is what a framework's "stream 0" handle means). */
int gbem_ctx_set_stream(gbem_ctx* ctx, void* cuda_stream);
/* Stream-ordered mode (on != 0): the device-pointer (_dev) calls enqueue their
 * work and return without blocking; the non-SPD pivot check of a factorisation
 * is latched and reported (GBEM_ENUMERIC, same message) by gbem_ctx_sync, which
 * synchronises the context's stream.  Off (default): every call is blocking and
 * reports its own errors, like the reference's exceptions. */
int gbem_ctx_set_async(gbem_ctx* ctx, int on);
int gbem_ctx_sync(gbem_ctx* ctx);
/* Number of this library's kernels launched on the context so far. */
int64_t gbem_ctx_launch_count(const gbem_ctx* ctx);

/* Batched u_pair_integral (kernels.hpp:270): out[k] = U(I_k, J_k), the
 * unnormalised integral (um^3); converged[k] (may be NULL) the Romberg flag.
 * Host buffers. */
int gbem_u_pair_integrals(gbem_ctx* ctx, const gbem_panels* I, const gbem_panels* J,
                          int64_t npairs, const gbem_quad_config* cfg, double* out,
                          int32_t* converged, gbem_assembly_stats* stats);

/* assemble_single (assembly.hpp:82): A[i][j] = U_ij / (|I_i||I_j|) for all
 * i <= j, mirrored.  The matrix stays on the device inside the context (n x n,
 * leading dimension = n) and feeds gbem_spd_solve; when A_host != NULL the full
 * symmetric matrix is also copied to A_host (row-major, lda >= n).
 * P: host arrays. */
int gbem_assemble_single(gbem_ctx* ctx, const gbem_panels* P, int64_t n,
                         const gbem_quad_config* cfg, double* A_host, int64_t lda,
                         gbem_assembly_stats* stats);
/* Same with device-resident panel arrays; no host synchronisation except to
 * read back stats when stats != NULL. */
int gbem_assemble_single_dev(gbem_ctx* ctx, const gbem_panels* P_dev, int64_t n,
                             const gbem_quad_config* cfg, gbem_assembly_stats* stats);
/* Row-block sharded assembly (no communication; rank r owns a work-balanced
 * row range): rows [row_begin, row_end) of the upper triangle into the caller's
 * device buffer, entry (i, j >= i) at out[(i - row_begin) * ld_out + j]
 * (ld_out >= n; entries j < i are not written). */
int gbem_assemble_rows_dev(gbem_ctx* ctx, const gbem_panels* P_dev, int64_t n,
                           int64_t row_begin, int64_t row_end, const gbem_quad_config* cfg,
                           double* out, int64_t ld_out, gbem_assembly_stats* stats);

/* As gbem_assemble_rows_dev but for complete rows (all j, the mirrored
 * entries recomputed locally): entry (i, j) at out[(i - row_begin) * ld_out + j].
 * This is the row block a sharded solver multiplies with. */
int gbem_assemble_rows_full_dev(gbem_ctx* ctx, const gbem_panels* P_dev, int64_t n,
                                int64_t row_begin, int64_t row_end, const gbem_quad_config* cfg,
                                double* out, int64_t ld_out, gbem_assembly_stats* stats);
/* Q = Ablk * P for a row block Ablk (rows x n, row i contiguous, leading
 * dimension ld) and P (n x K row-major: K values per panel, leading dimension
 * ldp >= K); Q is rows x K row-major with ldq >= K.  Device pointers. */
int gbem_rowblock_matvec_dev(gbem_ctx* ctx, const double* Ablk, int64_t ld, int64_t rows, int64_t n,
                             const double* P, int64_t ldp, int64_t K, double* Q, int64_t ldq);
/* Factor a device SPD matrix (column-major m x m, ldm) into the context and keep
 * the factor for repeated gbem_spd_solve_factored_dev calls (block-Jacobi
 * preconditioner of the sharded solver). */
int gbem_spd_factor_dev(gbem_ctx* ctx, const double* M, int64_t m, int64_t ldm, gbem_solve_stats* stats);
/* Y = A X with the context matrix (the original symmetric A: its preserved
 * strict upper triangle and diagonal, so also after a factorisation), X and Y
 * n x nrhs column-major on the device; the residual product of solver.hpp:47
 * (FP64 tensor cores for n >= 16,384). */
int gbem_matrix_apply_dev(gbem_ctx* ctx, const double* X, int64_t nrhs, double* Y);
int gbem_spd_solve_factored_dev(gbem_ctx* ctx, const double* B, int64_t nrhs, double* X, double* resid,
                                gbem_solve_stats* stats);

/* run_selftest (selftest.hpp:184-245, the CLI's `kernels selftest`): the
 * randomised audit of the pair evaluators against the brute-force oracle
 * (oracle.hpp:44-205), ten geometric classes x `pairs` seeded pairs, all on the
 * GPU (production single-layer evaluators, the double-layer kernel, and the
 * recursive oracle with Aitken extrapolation for touching classes).  Fills
 * cases[0..9]; *ncases = 10. */
typedef struct {
  char name[32];
  int32_t pairs;
  double worst_rel;
  double tol;
  int32_t pass;
  /* the worst pair: test and source panels (axis, level, a0, a1, b0, b1), the
   * source normal sign, the evaluator's and the oracle's values */
  double worst_test[6], worst_source[6];
  int32_t worst_nsign;
  double worst_value, worst_oracle;
} gbem_selftest_case;
int gbem_selftest(gbem_ctx* ctx, int32_t pairs, uint64_t seed, const gbem_quad_config* cfg,
                  gbem_selftest_case* cases, int32_t* ncases);
/* oracle_pair_integral (oracle.hpp:191-205) on the device for a pair list:
 * recursive dyadic subdivision to `depth` (0..6) with 6^4 Gauss leaves, the
 * single-layer kernel (double_layer = 0) or the double-layer one with source
 * normal signs nsign[k] (+1/-1; NULL = +1).  I, J: host arrays of npairs panels;
 * out: host, npairs values (um^3, like u_pair_integral). */
int gbem_oracle_pair_integrals(gbem_ctx* ctx, const gbem_panels* I, const gbem_panels* J, const int32_t* nsign,
                               int64_t npairs, int32_t double_layer, int32_t depth, double* out);

/* assemble_multi (assembly.hpp:110-175, replaces gbem::assemble_multi): the
 * Galerkin block system over all dielectric regions (double-layer
 * q_pair_integral kernels.hpp:295-315 and single-layer u_pair_integral with the
 * reference's reductions and Romberg rule, cfg = QuadratureConfig), same
 * panel / region arguments and outputs as gbem_assemble_collocation; the m x m
 * system stays in the context for gbem_lu_solve.  *all_converged ANDs the
 * kernels' convergence flags (assembly.hpp:97,133-135). */
int gbem_assemble_multi(gbem_ctx* ctx, const gbem_block_panels* P, int64_t n, const gbem_region* regions,
                        int32_t nregions, int32_t main_net, const gbem_quad_config* cfg, double* A_host, int64_t lda,
                        double* b_host, int64_t* m_out, int32_t* all_converged);

/* assemble_collocation (assembly.hpp:179-227): the point-collocation block
 * system of the scene for main net `main_net` (rows per region and boundary
 * panel, unknown map of assembly.hpp:51-75, closed-form u/q point kernels
 * kernels.hpp:319-355).  The m x m matrix stays in the context (gbem_lu_solve);
 * A_host (row-major, lda >= m) and b_host (m) receive copies when non-NULL.
 * *m_out = m.  GBEM_EINVAL for an unconstrained scene ("no Dirichlet
 * constraint anywhere in the scene (singular problem)"). */
int gbem_assemble_collocation(gbem_ctx* ctx, const gbem_block_panels* P, int64_t n,
                              const gbem_region* regions, int32_t nregions, int32_t main_net,
                              double* A_host, int64_t lda, double* b_host, int64_t* m_out);
/* lu_solve (solver.hpp:53-88) of the context matrix: LU with partial pivoting
 * (whole rows swapped), right-hand side b_host (m; NULL: the b of the last
 * gbem_assemble_collocation), solution x_host, relative residual
 * ||A x - b|| / ||b|| recomputed from the unfactored matrix.  A pivot below
 * 1e-14 max|A| -> GBEM_ENUMERIC "matrix numerically singular (smallest pivot
 * at row k)". */
int gbem_lu_solve(gbem_ctx* ctx, const double* b_host, double* x_host, double* resid, gbem_solve_stats* stats);
/* Upload a general (non-symmetric) matrix, row-major host with lda >= n, for
 * gbem_lu_solve. */
int gbem_matrix_upload_general(gbem_ctx* ctx, const double* A_host, int64_t n, int64_t lda);

/* Copy the assembled (or factored) matrix to the host: row-major, lda >= n. */
int gbem_matrix_download(gbem_ctx* ctx, double* A_host, int64_t lda);
/* Upload an arbitrary symmetric matrix (row-major host, lda >= n) as the
 * context's matrix, for solver tests independent of assembly. */
int gbem_matrix_upload(gbem_ctx* ctx, const double* A_host, int64_t n, int64_t lda);
/* Device pointer / leading dimension of the context matrix (column-major). */
int gbem_matrix_device(gbem_ctx* ctx, double** A_dev, int64_t* n, int64_t* lda);

/* cholesky_solve (solver.hpp:24) for nrhs right-hand sides: blocked Cholesky of
 * the context matrix with a DMMA trailing update, then two triangular solves.
 * B, X: host, column by column (B[r*n + i]).  resid (may be NULL) receives
 * ||A x_r - b_r|| / ||b_r|| recomputed from the original matrix.
 * Non-SPD: GBEM_ENUMERIC, message "matrix not positive definite (pivot at row k)". */
int gbem_spd_solve(gbem_ctx* ctx, const double* B, int64_t nrhs, double* X, double* resid,
                   gbem_solve_stats* stats);
/* Device-pointer variant; resid_dev may be NULL. */
int gbem_spd_solve_dev(gbem_ctx* ctx, const double* B_dev, int64_t nrhs, double* X_dev,
                       double* resid_dev, gbem_solve_stats* stats);

/* net_charges (extraction.hpp:55-79) for the K-RHS system: with net_of_panel[p]
 * in [0, K) for conductor panels and -1 otherwise (e.g. grounded outer panels),
 * C[r*K + k] = scale * sum_{p : net_of_panel[p] == k} X[r*n + p], and
 * outer[r] (may be NULL) the sum over panels with net -1.  scale = eps_r*eps0*1e-6.
 * Device pointers. */
int gbem_net_charges_dev(gbem_ctx* ctx, const int32_t* net_of_panel, int64_t n,
                         const double* X, int64_t nrhs, int32_t K, double scale, double* C,
                         double* outer);

/* Capacitance matrix of a single-dielectric panel set in one call (the shared
 * K-right-hand-side path of capacitance_matrix, extraction.hpp:162-184):
 * assemble, factor, solve with B[:, r] = 1 on the panels of net r, and reduce
 * C[r*K + k] = eps_r * eps0 * 1e-6 * sum_{p in net k} X[p, r] (farads).
 * net_of_panel[p] in [0, K) for conductor panels, -1 for grounded outer panels.
 * Host buffers (every host<->device copy happens inside the call).  With several
 * ranks attached to the context (gbem_ctx_init_nccl / gbem_ctx_set_collectives)
 * every rank calls it and the solve runs on row-block shards
 * (gbem_pcg_extract_cmatrix, Jacobi blocks of ~12k rows); sstats is then zeroed. */
int gbem_extract_cmatrix(gbem_ctx* ctx, const gbem_panels* P, int64_t n, const int32_t* net_of_panel,
                         int32_t K, double eps_r, const gbem_quad_config* cfg, double* C, double* resid,
                         gbem_assembly_stats* astats, gbem_solve_stats* sstats);
/* Device-pointer variant (panels, net_of_panel, C, resid on the device); runs
 * stream-ordered and only synchronises to read back stats when requested. */
int gbem_extract_cmatrix_dev(gbem_ctx* ctx, const gbem_panels* P, int64_t n, const int32_t* net_of_panel,
                             int32_t K, double eps_r, const gbem_quad_config* cfg, double* C, double* resid,
                             gbem_assembly_stats* astats, gbem_solve_stats* sstats);

/* Diagnostic: fill the shared memory of every SM with `value` (one maximal
 * CTA per SM).  Tests use it to prove that no kernel reads shared memory it
 * did not write (e.g. NaN left by an earlier kernel). */
int gbem_debug_fill_shared(gbem_ctx* ctx, double value);

/* ------------------------------------------------------------------------
 * Row-block sharded solve (no reference counterpart: the
 * reference solves with dense Cholesky only, solver.hpp:24-50).  When the
 * matrix does not fit one GPU, rank r of P holds complete rows
 * [r*m, min((r+1)*m, n)) of A, m = ceil(n / P), assembled locally with no
 * communication, and A X = B is solved by block-Jacobi preconditioned CG
 * (K recurrences sharing every launch and collective).  Per iteration: an
 * all-gather of the search directions (n x K), the local DMMA product
 * A_r P, two all-reduces of K-vectors, and the preconditioner as one DMMA
 * GEMM against the explicit inverse of each Jacobi block.
 *
 * Collectives: the context owns an NCCL communicator (gbem_ctx_init_nccl;
 * libnccl.so.2 is loaded at run time, so a process that already holds NCCL,
 * e.g. through torch, shares it), or the host plugs its own (MPI, gloo ...)
 * through gbem_collectives.  With one rank no collective is issued. */
#define GBEM_NCCL_UNIQUE_ID_BYTES 128
/* ncclGetUniqueId: rank 0 calls it and distributes the 128 bytes out of band. */
int gbem_nccl_unique_id(void* id_out);
/* Attach an NCCL communicator of nranks ranks (ncclCommInitRank) to ctx. */
int gbem_ctx_init_nccl(gbem_ctx* ctx, int32_t nranks, int32_t rank, const void* id);

/* Host-provided collectives on device buffers of doubles, called on the
 * calling thread with the context's cudaStream_t; each returns 0 on success.
 *   all_gather: every rank contributes `count` doubles, recv holds nranks*count
 *               in rank order;
 *   all_reduce_sum: in-place sum of `count` doubles. */
typedef struct {
  void* user;
  int (*all_gather)(void* user, const double* send, double* recv, int64_t count, void* stream);
  int (*all_reduce_sum)(void* user, double* buf, int64_t count, void* stream);
} gbem_collectives;
int gbem_ctx_set_collectives(gbem_ctx* ctx, int32_t nranks, int32_t rank, const gbem_collectives* coll);

typedef struct {
  double tol;              /* stop a column at ||b - A x|| / ||b|| <= tol (default 1e-10) */
  int32_t max_iter;        /* default 1000 */
  int32_t jacobi_blocks;   /* Jacobi blocks per rank (default 1: the rank's diagonal block) */
} gbem_pcg_options;

typedef struct {
  int64_t n, rows_local, row_begin;
  int32_t nranks, rank, iterations, converged;
  double max_rel_resid;     /* max over columns of ||B - A X|| / ||B||, recomputed from A at the end */
  double ms_assembly, ms_precond, ms_iterations, ms_matvec, ms_total;
  double matvec_flops;      /* 2 rows n K per product, summed over the products of this rank */
} gbem_pcg_stats;

/* C-matrix extraction on row-block shards: every rank calls it with the same
 * (replicated) panels and net_of_panel (net -1: grounded outer panels); C (K x K),
 * resid (K) and outer (K: the charge on the net -1 panels per row, may be NULL)
 * come out identical on every rank.  Device pointers; the _dev variant is
 * stream-ordered apart from the convergence polling. */
int gbem_pcg_extract_cmatrix_dev(gbem_ctx* ctx, const gbem_panels* P_dev, int64_t n,
                                 const int32_t* net_of_panel, int32_t K, double eps_r,
                                 const gbem_quad_config* cfg, const gbem_pcg_options* opt,
                                 double* C, double* resid, double* outer, gbem_assembly_stats* astats,
                                 gbem_pcg_stats* pstats);
/* Host-buffer variant (panels, net_of_panel, C, resid, outer in host memory). */
int gbem_pcg_extract_cmatrix(gbem_ctx* ctx, const gbem_panels* P, int64_t n, const int32_t* net_of_panel,
                             int32_t K, double eps_r, const gbem_quad_config* cfg, const gbem_pcg_options* opt,
                             double* C, double* resid, double* outer, gbem_assembly_stats* astats,
                             gbem_pcg_stats* pstats);
/* Ranks attached to the context (1 until gbem_ctx_init_nccl / gbem_ctx_set_collectives). */
int32_t gbem_ctx_nranks(const gbem_ctx* ctx);
int32_t gbem_ctx_rank(const gbem_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif

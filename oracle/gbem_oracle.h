/* gbem_oracle.h — TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * Plain-C restatement of the reference GBEM single-layer hot path, used as the
 * parity checker for the B200 kernels.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Parity pinned against: the frozen single-layer values of
 * proj/tests/test_kernels.cpp:166-215, the oracle values of
 * proj/tests/test_oracle.cpp:60-88, the Romberg/t^4 cases of
 * proj/tests/test_quadrature.cpp:11-79 and, pair by pair, against the
 * reference headers themselves compiled into oracle/_ref (see oracle/Makefile).
 */
#ifndef GBEM_ORACLE_H
#define GBEM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Rect (proj/include/gbem/geometry.hpp:52-76): plane x[axis] == level,
 * span a / span b along the in-plane axes in axis-index order. */
typedef struct {
  int axis;
  double level;
  double a0, a1, b0, b1;
} orc_rect;

/* KernelValue (kernels.hpp:16-20). status: 0 ok, 2 non-finite sample
 * (the reference throws NumericalError there, quadrature.hpp:34-35,46). */
typedef struct {
  double value;
  int converged;
  long evals;
  int status;
} orc_kv;

/* u_pair_integral (kernels.hpp:270-291) with QuadratureConfig{relTol,maxLevels}
 * (quadrature.hpp:12-15). */
orc_kv orc_u_pair_integral(const orc_rect* Ii, const orc_rect* Ij, double rel_tol,
                           int max_levels);

/* Batched form over pair lists (one thread per pair block when nthreads > 1). */
int orc_u_pairs(int64_t npairs, const orc_rect* a, const orc_rect* b, double rel_tol,
                int max_levels, double* out, int* converged, int nthreads);

/* Composite tensor 6-point Gauss (the rule of oracle.hpp:45-81 with the nodes of
 * quadrature.hpp:116-124) with each panel split sub x sub: the far-field
 * "truth" of SURVEY §8(c). */
double orc_gauss_pair(const orc_rect* r1, const orc_rect* r2, int sub);

/* oracle_pair_integral(SingleLayer, ...) restated (oracle.hpp:105-131,191-205). */
double orc_oracle_pair_integral(const orc_rect* Ii, const orc_rect* Ij, int depth);

/* Gap between the closed world extents (rectDistance, geometry.hpp:79-87) and
 * diameter (geometry.hpp:73). */
double orc_rect_distance(const orc_rect* a, const orc_rect* b);
double orc_rect_diameter(const orc_rect* a);

/* assemble_single (assembly.hpp:82-104) on a panel list: A is n x n row-major,
 * A[i][j] = A[j][i] = U_ij / (|I_i||I_j|).  Returns 0, or 2 on a non-finite
 * sample; *all_converged receives the AND of the converged flags. */
int orc_assemble_single(int64_t n, const orc_rect* p, double rel_tol, int max_levels,
                        double* A, int* all_converged, int nthreads);

/* cholesky_solve (solver.hpp:24-50) in the reference's loop order, on row-major
 * A (n x n) for nrhs right-hand sides stored column by column (B[r*n + i]).
 * Returns 0, 1 on bad dims, 2 with *bad_pivot = k for "matrix not positive
 * definite (pivot at row k)".  resid[r] = ||A x - b|| / ||b|| (solver.hpp:17-21). */
int orc_cholesky_solve(int64_t n, const double* A, int64_t nrhs, const double* B, double* X,
                       double* resid, int64_t* bad_pivot);

/* u_point_rect / q_point_rect (kernels.hpp:319-355): closed-form single- and
 * double-layer potentials of a unit density on R at the point x; nsign is
 * R.normalSign. */
double orc_u_point_rect(const double x[3], const orc_rect* R);
double orc_q_point_rect(const double x[3], const orc_rect* R, int nsign);

/* assemble_collocation (assembly.hpp:179-227) on flat class-contiguous panel
 * arrays (kind 0 conductor, 1 dirichlet outer, 2 neumann outer, 3 interface),
 * regions (id, eps) in any order.  A is m x m row-major (m = *m_out, caller
 * buffer of at least (panels + interfaces)^2), b has m entries.  Returns 0, 1
 * for invalid input (no Dirichlet constraint / unknown region), 2 for a
 * non-square system. */
int orc_assemble_collocation(int64_t n, const orc_rect* p, const int* nsign, const int* kind, const int* net,
                             const int* reg_a, const int* reg_b, int nreg, const int* reg_id,
                             const double* reg_eps, int main_net, double* A, double* b, int64_t* m_out);

/* q_pair_integral (kernels.hpp:295-315): test Ii, source Ij with normal sign nsign_j. */
orc_kv orc_q_pair_integral(const orc_rect* Ii, const orc_rect* Ij, int nsign_j, double rel_tol, int max_levels);

/* assemble_multi (assembly.hpp:110-175), same arguments and layout as
 * orc_assemble_collocation plus the QuadratureConfig; returns 3 on a non-finite
 * integrand sample; *all_converged ANDs the kernels' flags. */
int orc_assemble_multi(int64_t n, const orc_rect* p, const int* nsign, const int* kind, const int* net,
                       const int* reg_a, const int* reg_b, int nreg, const int* reg_id, const double* reg_eps,
                       int main_net, double rel_tol, int max_levels, double* A, double* b, int64_t* m_out,
                       int* all_converged);

/* lu_solve (solver.hpp:53-88): partial pivoting with whole-row swaps on a
 * row-major copy of A (n x n).  Returns 0, or 2 with *bad_row = k for "matrix
 * numerically singular (smallest pivot at row k)".  *resid = ||A x - b|| / ||b||. */
int orc_lu_solve(int64_t n, const double* A, const double* b, double* x, double* resid, int64_t* bad_row);

/* Romberg / integrateSegment on test integrands (quadrature.hpp:27-113), for the
 * known-answer cases of test_quadrature.cpp. which: 0 x^2, 1 const 1, 2 log1p,
 * 3 x (empty interval), 4 sin, 5 1/x, 6 1/sqrt(x), 7 log x, 8 1/sqrt(1-x),
 * 9 1/sqrt(x)+1/sqrt(1-x), 10 1/sqrt(|x|), 11 x^2 (splits). mode: 0 romberg,
 * 1 integrateSegment(singA, singB), 2 integrateWithSplits. */
double orc_quad_test(int which, int mode, double a, double b, int singA, int singB,
                     int* status, int* converged, long* evals);

/* solver.hpp:28-37 factor loop with Eigen's column-major L (timing of the
 * reference's CPU order; bench.py cpu_baseline / --impl reference). */
int orc_cholesky_factor_colmajor(int64_t n, const double* A, double* L, int64_t* bad_pivot);

#ifdef __cplusplus
}
#endif
#endif

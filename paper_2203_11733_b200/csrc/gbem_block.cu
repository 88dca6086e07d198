// gbem_block.cu — the block (mixed-unknown) system of the reference on B200:
// point-collocation assembly and the dense LU solve with partial pivoting.
//
//   assemble_collocation (proj/include/gbem/assembly.hpp:179-227) with the
//   closed-form point kernels u_point_rect / q_point_rect (kernels.hpp:319-355)
//   -> gbem_assemble_collocation: one warp per system row (region, panel);
//   lu_solve (solver.hpp:53-88) -> gbem_lu_solve: blocked right-looking LU,
//   NB = 64, pivot search / row swap / panel update in a cooperative kernel
//   (three grid barriers per column, whole rows swapped as the reference does,
//   b included), U12 = inv(L11) A12 by per-column substitution, the O(n^3)
//   trailing update A22 -= L21 U12 on the DMMA GEMM (k_gemm_g<kSub, NN>), then a
//   cooperative forward/backward substitution; residual ||A x - b|| / ||b||
//   from a preserved copy of A (solver.hpp:17-21).
//   Singular matrix: |pivot| < 1e-14 max|A| -> GBEM_ENUMERIC "matrix
//   numerically singular (smallest pivot at row k)", as solver.hpp:68-70.
#include <algorithm>
#include <cmath>
#include <vector>

#include <cooperative_groups.h>

#include "gbem_common.cuh"
#include "gbem_ctx.cuh"
#include "gbem_dmma_gemm.cuh"
#include "gbem_near.cuh"

namespace cg = cooperative_groups;
using namespace gbem_gpu;

namespace {

// ------------------------------------------------------------ point kernels

// u_point_rect (kernels.hpp:319-338): single-layer potential of a unit density
// on R at x (closed form, corner sum of mulLog terms minus h atan).
__device__ double d_u_point_rect(const double x[3], const DPanel& R) {
  const int i0 = ip0(R.axis), i1 = ip1(R.axis);
  const double h = x[R.axis] - R.level;
  const double u1 = R.a0 - x[i0], u2 = R.a1 - x[i0];
  const double v1 = R.b0 - x[i1], v2 = R.b1 - x[i1];
  const double scale = fmax(fmax(fmax(fabs(u1), fabs(u2)), fmax(fabs(v1), fabs(v2))), fmax(fabs(h), 1e-30));
  const double guard = 1e-14 * scale;
  const double h2 = h * h;
  auto F = [&](double u, double v) {
    double t = d_mul_log(v, u, v * v + h2, guard) + d_mul_log(u, v, u * u + h2, guard);
    if (h != 0.0) {
      const double r = sqrt(u * u + v * v + h2);
      t -= h * atan(u * v / (h * r));
    }
    return t;
  };
  return (F(u2, v2) - F(u1, v2) - F(u2, v1) + F(u1, v1)) / kFourPi;
}

// q_point_rect (kernels.hpp:342-355): signed solid-angle fraction; 0 in-plane.
__device__ double d_q_point_rect(const double x[3], const DPanel& R, int nsign) {
  const double h = x[R.axis] - R.level;
  if (h == 0.0) return 0.0;
  const int i0 = ip0(R.axis), i1 = ip1(R.axis);
  const double u1 = R.a0 - x[i0], u2 = R.a1 - x[i0];
  const double v1 = R.b0 - x[i1], v2 = R.b1 - x[i1];
  const double h2 = h * h;
  auto G = [&](double u, double v) {
    const double r = sqrt(u * u + v * v + h2);
    return atan(u * v / (h * r));
  };
  const double sum = G(u2, v2) - G(u1, v2) - G(u2, v1) + G(u1, v1);
  return (double)nsign * sum / kFourPi;
}

// Block-system panel: geometry + the attributes the coefficients need.
struct BPanel {
  DPanel g;
  int nsign, kind, rega, regb;
  int qcol, ucol;
  double area, known;  // knownPotential (assembly.hpp:42-44)
};

// One warp per row (region r, panel a) of assemble_collocation
// (assembly.hpp:205-221), test point = the centroid of panel a:
//   coefU = q_point_rect(x, P_c) sideSign(P_c, r) + 1/2 [c == a]
//           -> A(row, uCol[c]) or b(row) -= coefU * known(c);
//   coefX = -u_point_rect(x, P_c) / |P_c| (x -(eps_A/eps_r) on the B side of an
//           interface) -> A(row, qCol[c]), skipped for Neumann panels.
// Each (row, c) writes distinct columns, so A needs no atomics; b is a warp sum.
__global__ void k_collocation(const BPanel* __restrict__ P, const int32_t* __restrict__ row_region,
                              const int32_t* __restrict__ row_panel, const int32_t* __restrict__ list_off,
                              const int32_t* __restrict__ list, const int32_t* __restrict__ region_ids,
                              const double* __restrict__ region_eps, int nreg, int m, double* A, long long lda,
                              double* b) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= m) return;
  const int ri = row_region[warp], a = row_panel[warp];
  const int rid = region_ids[ri];
  const double eps_r = region_eps[ri];
  const BPanel pa = P[a];
  double x[3];
  for (int k = 0; k < 3; ++k) {
    double lo, hi;
    panel_extent(pa.g, k, lo, hi);
    x[k] = 0.5 * (lo + hi);  // Rect::center
  }
  double bsum = 0.0;
  for (int t = list_off[ri] + lane; t < list_off[ri + 1]; t += 32) {
    const int c = list[t];
    const BPanel pc = P[c];
    const double side = pc.kind == 3 ? (pc.rega == rid ? 1.0 : -1.0) : -1.0;  // sideSign (assembly.hpp:37-40)
    const double coefU = d_q_point_rect(x, pc.g, pc.nsign) * side + (c == a ? 0.5 : 0.0);
    if (pc.ucol >= 0)
      A[(long long)pc.ucol * lda + warp] += coefU;
    else
      bsum -= coefU * pc.known;
    if (pc.kind == 2) continue;  // Neumann: q known zero
    double coefX = -d_u_point_rect(x, pc.g) / pc.area;
    if (pc.kind == 3 && pc.regb == rid) {
      double eps_a = 1.0;
      for (int k = 0; k < nreg; ++k)
        if (region_ids[k] == pc.rega) eps_a = region_eps[k];
      coefX *= -(eps_a / eps_r);
    }
    A[(long long)pc.qcol * lda + warp] += coefX;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) bsum += __shfl_xor_sync(0xffffffffu, bsum, off);
  if (lane == 0) b[warp] = bsum;
}

// Galerkin block system (assemble_multi, assembly.hpp:110-175): one warp per
// (row, c) of a region's local blocks; the warp evaluates the reference's
// double-layer q_pair_integral(P_a, P_c) and single-layer u_pair_integral with
// the reference's own reductions and warp-cooperative Romberg (gbem_near.cuh):
//   coefU = Qloc(a, c) / |P_a| + 1/2 [c == a],  Qloc = q * nsign_c * sideSign(P_c, region)
//           -> A(row, uCol[c]) or b(row) -= coefU * known(c);
//   coefX = -Uloc(a, c) / (|P_a| |P_c|) (x -(eps_A / eps_r) on the B side of an
//           interface) -> A(row, qCol[c]), skipped for Neumann panels.
// A's (row, column) entries are written once each; b accumulates atomically.
// flags[0] counts non-converged Romberg runs, flags[1] non-finite samples.
__global__ void __launch_bounds__(128)
    k_galerkin_multi(const BPanel* __restrict__ P, const int32_t* __restrict__ row_region,
                     const int32_t* __restrict__ row_panel, const int32_t* __restrict__ list_off,
                     const int32_t* __restrict__ list, const int32_t* __restrict__ region_ids,
                     const double* __restrict__ region_eps, int nreg, double* A, long long lda, double* b,
                     double rel_tol, int max_levels, unsigned long long* flags) {
  const int row = blockIdx.y, lane = threadIdx.x & 31;
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int ri = row_region[row], a = row_panel[row];
  const int lo = list_off[ri], hi = list_off[ri + 1];
  if (lo + t >= hi) return;  // warp-uniform
  const int c = list[lo + t];
  const int rid = region_ids[ri];
  const double eps_r = region_eps[ri];
  const BPanel pa = P[a], pc = P[c];
  WarpQuad st;
  double q = 0.0;
  if (pa.g.axis != pc.g.axis)
    q = warp_q_orthogonal(pa.g, pc.g, rel_tol, max_levels, lane, st);
  else if (pa.g.level != pc.g.level)
    q = warp_q_parallel(pa.g, pc.g, rel_tol, max_levels, lane, st);
  q *= (double)pc.nsign;
  const double side = pc.kind == 3 ? (pc.rega == rid ? 1.0 : -1.0) : -1.0;  // sideSign (assembly.hpp:37-40)
  const double coefU = q * side / pa.area + (c == a ? 0.5 : 0.0);
  if (lane == 0) {
    if (pc.ucol >= 0)
      A[(long long)pc.ucol * lda + row] = coefU;
    else if (pc.known != 0.0)
      atomicAdd(&b[row], -coefU * pc.known);
  }
  if (pc.kind != 2) {  // Neumann: q known zero
    // u_pair_integral (kernels.hpp:270-291): canonical argument order
    const bool sw = d_rect_less(pc.g, pa.g);
    const DPanel& x = sw ? pc.g : pa.g;
    const DPanel& y = sw ? pa.g : pc.g;
    double U;
    if (x.axis == y.axis)
      U = x.level == y.level ? d_u_coplanar(x.a0, x.a1, x.b0, x.b1, y.a0, y.a1, y.b0, y.b1)
                             : warp_u_parallel(x, y, rel_tol, max_levels, lane, st);
    else
      U = warp_u_orthogonal(x, y, rel_tol, max_levels, lane, st);
    double coefX = -U / (pa.area * pc.area);
    if (pc.kind == 3 && pc.regb == rid) {
      double eps_a = 1.0;
      for (int k = 0; k < nreg; ++k)
        if (region_ids[k] == pc.rega) eps_a = region_eps[k];
      coefX *= -(eps_a / eps_r);
    }
    if (lane == 0) A[(long long)pc.qcol * lda + row] = coefX;
  }
  if (lane == 0) {
    if (!st.converged) atomicAdd(&flags[0], 1ull);
    if (st.nonfinite) atomicAdd(&flags[1], 1ull);
  }
}

// ------------------------------------------------------------ LU

constexpr int LNB = 64;          // LU block size
constexpr int kLuThreads = 256;

__device__ __forceinline__ void argmax_merge(double& v, int& r, double v2, int r2) {
  if (v2 > v || (v2 == v && r2 < r)) {
    v = v2;
    r = r2;
  }
}

// Panel factorisation with partial pivoting of columns [k0, k0 + nb), whole
// rows swapped (and b).  part: 2 * gridDim.x scratch; info: first bad pivot.
__global__ void __launch_bounds__(kLuThreads, 1)
    k_lu_panel(double* A, long long lda, int m, int k0, int nb, double* b, int* piv, double thresh, double* part,
               int* info) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sv[kLuThreads / 32];
  __shared__ int sr[kLuThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long gtid = grid.thread_rank(), gsz = grid.size();
  for (int j = k0; j < k0 + nb; ++j) {
    // 1. argmax |A(r, j)|, r >= j (first index on ties, like Eigen's maxCoeff)
    double v = -1.0;
    int r = m;
    for (long long rr = j + gtid; rr < m; rr += gsz) argmax_merge(v, r, fabs(A[(long long)j * lda + rr]), (int)rr);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, v, off);
      const int r2 = __shfl_xor_sync(0xffffffffu, r, off);
      argmax_merge(v, r, v2, r2);
    }
    if (lane == 0) {
      sv[warp] = v;
      sr[warp] = r;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < kLuThreads / 32; ++w) argmax_merge(v, r, sv[w], sr[w]);
      part[2 * blockIdx.x] = v;
      part[2 * blockIdx.x + 1] = (double)r;  // exact: r < 2^31
    }
    grid.sync();
    // every block folds the partials in the same order: one deterministic pivot
    v = -1.0;
    r = m;
    for (unsigned q = 0; q < gridDim.x; ++q) argmax_merge(v, r, part[2 * q], (int)part[2 * q + 1]);
    const int p = r;
    if (gtid == 0) {
      piv[j] = p;
      if (!(v >= thresh)) atomicMin(info, j);
    }
    // 2. swap rows j and p over all columns, and b
    if (p != j && p < m) {
      for (long long c = gtid; c < m; c += gsz) {
        const double t = A[c * lda + j];
        A[c * lda + j] = A[c * lda + p];
        A[c * lda + p] = t;
      }
      if (gtid == 0) {
        const double t = b[j];
        b[j] = b[p];
        b[p] = t;
      }
    }
    grid.sync();
    // 3. multipliers f = A(r, j) / A(j, j) and the in-panel rank-1 update
    double d = A[(long long)j * lda + j];
    if (d == 0.0) d = 1.0;  // singular: flagged above, keep the arithmetic finite
    for (long long rr = j + 1 + gtid; rr < m; rr += gsz) {
      const double f = A[(long long)j * lda + rr] / d;
      A[(long long)j * lda + rr] = f;
      for (int c = j + 1; c < k0 + nb; ++c) A[(long long)c * lda + rr] -= f * A[(long long)c * lda + j];
    }
    grid.sync();
  }
}

// U12 = inv(L11) A12 (unit lower L11 = A[k0.., k0..] below the diagonal), one
// thread per column of A12, the column's LNB values in registers.
__global__ void __launch_bounds__(128)
    k_lu_trsm(double* A, long long lda, int m, int k0, int nb) {
  __shared__ double L[LNB][LNB + 1];
  for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
    const int r = idx % nb, c = idx / nb;
    L[r][c] = A[(long long)(k0 + c) * lda + k0 + r];
  }
  __syncthreads();
  const long long col = (long long)k0 + nb + blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= m) return;
  double* x = A + col * lda + k0;
  double v[LNB];
#pragma unroll
  for (int i = 0; i < LNB; ++i) v[i] = i < nb ? x[i] : 0.0;
#pragma unroll
  for (int l = 0; l < LNB; ++l)
#pragma unroll
    for (int i = l + 1; i < LNB; ++i)
      if (i < nb) v[i] = fma(-L[i][l], v[l], v[i]);
#pragma unroll
  for (int i = 0; i < LNB; ++i)
    if (i < nb) x[i] = v[i];
}

// Forward (unit L) and backward (U) substitution, one grid barrier per 64-row
// block; the block triangle is solved by warp 0 of every CTA (redundantly),
// the other rows are updated column-by-column (coalesced along the rows).
// w: permuted b, updated below each block; z: forward result, updated above
// each block in the backward sweep; x: solution.  Solved blocks go to the next
// array, so no CTA reads a value another CTA rewrites in the same step.
__global__ void __launch_bounds__(kLuThreads, 1)
    k_lu_solve(const double* __restrict__ A, long long lda, int m, double* w, double* z, double* x) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double yb[LNB];
  const int tid = threadIdx.x, lane = tid & 31;
  const long long gtid = grid.thread_rank(), gsz = grid.size();
  const int nblk = (m + LNB - 1) / LNB;
  for (int bb = 0; bb < nblk; ++bb) {
    const int r0 = bb * LNB, nb = min(LNB, m - r0);
    if (tid < 32) {
      double v0 = lane < nb ? w[r0 + lane] : 0.0, v1 = lane + 32 < nb ? w[r0 + lane + 32] : 0.0;
      for (int j = 0; j < nb; ++j) {
        const double yj = __shfl_sync(0xffffffffu, j < 32 ? v0 : v1, j & 31);
        const double l0 = lane > j && lane < nb ? A[(long long)(r0 + j) * lda + r0 + lane] : 0.0;
        const double l1 = lane + 32 > j && lane + 32 < nb ? A[(long long)(r0 + j) * lda + r0 + lane + 32] : 0.0;
        v0 = fma(-l0, yj, v0);
        v1 = fma(-l1, yj, v1);
      }
      if (lane < nb) yb[lane] = v0;
      if (lane + 32 < nb) yb[lane + 32] = v1;
    }
    __syncthreads();
    if (blockIdx.x == 0)
      for (int i = tid; i < nb; i += blockDim.x) z[r0 + i] = yb[i];
    for (long long r = r0 + nb + gtid; r < m; r += gsz) {
      double s = 0.0;
      for (int c = 0; c < nb; ++c) s = fma(A[(long long)(r0 + c) * lda + r], yb[c], s);
      w[r] -= s;
    }
    grid.sync();
  }
  for (int bb = nblk - 1; bb >= 0; --bb) {
    const int r0 = bb * LNB, nb = min(LNB, m - r0);
    if (tid < 32) {
      double v0 = lane < nb ? z[r0 + lane] : 0.0, v1 = lane + 32 < nb ? z[r0 + lane + 32] : 0.0;
      for (int j = nb - 1; j >= 0; --j) {
        const double ujj = A[(long long)(r0 + j) * lda + r0 + j];
        if (lane == (j & 31)) {  // x_j = (z_j - sum_{l > j} U(j, l) x_l) / U(j, j)
          if (j < 32) v0 /= ujj;
          else v1 /= ujj;
        }
        const double xj = __shfl_sync(0xffffffffu, j < 32 ? v0 : v1, j & 31);
        const double u0 = lane < j ? A[(long long)(r0 + j) * lda + r0 + lane] : 0.0;
        const double u1 = lane + 32 < j ? A[(long long)(r0 + j) * lda + r0 + lane + 32] : 0.0;
        v0 = fma(-u0, xj, v0);
        v1 = fma(-u1, xj, v1);
      }
      if (lane < nb) yb[lane] = v0;
      if (lane + 32 < nb) yb[lane + 32] = v1;
    }
    __syncthreads();
    if (blockIdx.x == 0)
      for (int i = tid; i < nb; i += blockDim.x) x[r0 + i] = yb[i];
    for (long long r = gtid; r < r0; r += gsz) {
      double s = 0.0;
      for (int c = 0; c < nb; ++c) s = fma(A[(long long)(r0 + c) * lda + r], yb[c], s);
      z[r] -= s;
    }
    grid.sync();
  }
}

// r = A0 x - b0 row sums, then ||r|| / ||b0|| (solver.hpp:17-21), one block.
__global__ void k_gemv_resid(const double* __restrict__ A0, long long lda, int m, const double* __restrict__ x,
                             const double* __restrict__ b0, double* r) {
  const long long row = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (row >= m) return;
  double s = 0.0;
  for (int c = 0; c < m; ++c) s = fma(A0[(long long)c * lda + row], x[c], s);
  r[row] = s - b0[row];
}

__global__ void k_norm_ratio(const double* __restrict__ r, const double* __restrict__ b0, int m, double* out) {
  __shared__ double s1[256], s2[256];
  double a = 0.0, c = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    a = fma(r[i], r[i], a);
    c = fma(b0[i], b0[i], c);
  }
  s1[threadIdx.x] = a;
  s2[threadIdx.x] = c;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      s1[threadIdx.x] += s1[threadIdx.x + w];
      s2[threadIdx.x] += s2[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double bn = sqrt(s2[0]);
    out[0] = sqrt(s1[0]) / (bn > 0.0 ? bn : 1.0);
  }
}

__global__ void k_absmax(const double* __restrict__ A, long long lda, int m, unsigned long long* out) {
  double v = 0.0;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)m * m;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long c = idx / m, r = idx % m;
    v = fmax(v, fabs(A[c * lda + r]));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(v));  // v >= 0: bits order
}

}  // namespace

// Host side of the block system: unknown map (assembly.hpp:46-75), rows per
// region (partition.hpp:238-243), device arrays, the collocation kernel.
int gbem_internal_assemble_block(gbem_ctx* ctx, const gbem_block_panels* P, int64_t n, const gbem_region* regions,
                                 int32_t nreg, int32_t main_net, bool galerkin, const gbem_quad_config* cfg,
                                 int64_t* m_out, int64_t* nonconv_out) {
  if (n <= 0 || nreg <= 0) return ctx->fail(GBEM_EINVAL, "empty block system");
  if (!P || !P->kind || !P->net || !P->reg_a || !P->reg_b || !P->nsign || !P->geom.axis || !P->geom.level ||
      !P->geom.a_lo || !P->geom.a_hi || !P->geom.b_lo || !P->geom.b_hi || !regions)
    return ctx->fail(GBEM_EINVAL, "null block-panel array");
  const int32_t* kind = P->kind;
  for (int64_t k = 1; k < n; ++k)
    if (kind[k] < kind[k - 1]) return ctx->fail(GBEM_EINVAL, "panels must be class-contiguous (partition.hpp:48-51)");
  int64_t off[5] = {0, 0, 0, 0, 0};
  for (int64_t k = 0; k < n; ++k) {
    if (kind[k] < 0 || kind[k] > 3) return ctx->fail(GBEM_EINVAL, "panel kind must be 0..3");
    off[kind[k] + 1]++;
  }
  for (int k = 1; k < 5; ++k) off[k] += off[k - 1];
  if (off[2] == 0)  // no conductor and no Dirichlet outer panel (assembly.hpp:188-189)
    return ctx->fail(GBEM_EINVAL, "no Dirichlet constraint anywhere in the scene (singular problem)");
  // buildUnknownMap (assembly.hpp:51-75)
  std::vector<BPanel> bp((size_t)n);
  const int64_t o3 = off[3];
  for (int64_t p = 0; p < n; ++p) {
    BPanel& b = bp[(size_t)p];
    b.g.level = P->geom.level[p];
    b.g.a0 = P->geom.a_lo[p];
    b.g.a1 = P->geom.a_hi[p];
    b.g.b0 = P->geom.b_lo[p];
    b.g.b1 = P->geom.b_hi[p];
    b.g.axis = P->geom.axis[p];
    b.g.pad = 0;
    if (b.g.axis > 2 || !(b.g.a0 < b.g.a1) || !(b.g.b0 < b.g.b1))
      return ctx->fail(GBEM_EINVAL, "bad panel geometry (panel " + std::to_string(p) + ")");
    b.nsign = P->nsign[p] >= 0 ? 1 : -1;
    b.kind = kind[p];
    b.rega = P->reg_a[p];
    b.regb = P->reg_b[p];
    b.area = (b.g.a1 - b.g.a0) * (b.g.b1 - b.g.b0);
    b.known = (kind[p] == 0 && P->net[p] == main_net) ? 1.0 : 0.0;  // knownPotential
    b.qcol = b.ucol = -1;
    if (kind[p] == 0 || kind[p] == 1)
      b.qcol = (int)p;
    else if (kind[p] == 2)
      b.ucol = (int)p;
    else {
      const int64_t t = p - o3;
      b.ucol = (int)(o3 + 2 * t);
      b.qcol = (int)(o3 + 2 * t + 1);
    }
  }
  const int64_t cols = o3 + 2 * (off[4] - o3);
  // regionPanels (partition.hpp:238-243), ascending region id; rows in that order
  std::vector<int> order(nreg);
  for (int k = 0; k < nreg; ++k) order[k] = k;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return regions[a].id < regions[b].id; });
  std::vector<int32_t> ids(nreg), list_off(nreg + 1, 0), list, row_region, row_panel;
  std::vector<double> eps(nreg);
  for (int k = 0; k < nreg; ++k) {
    ids[k] = regions[order[k]].id;
    eps[k] = regions[order[k]].eps;
  }
  for (int64_t p = 0; p < n; ++p) {
    bool found = false;
    for (int k = 0; k < nreg; ++k) found |= bp[(size_t)p].rega == ids[k];
    if (!found) return ctx->fail(GBEM_EINVAL, "panel references unknown region");
  }
  for (int k = 0; k < nreg; ++k) {
    list_off[k] = (int32_t)list.size();
    for (int64_t p = 0; p < n; ++p)
      if (bp[(size_t)p].rega == ids[k] || (bp[(size_t)p].kind == 3 && bp[(size_t)p].regb == ids[k]))
        list.push_back((int32_t)p);
    for (int32_t t = list_off[k]; t < (int32_t)list.size(); ++t) {
      row_region.push_back(k);
      row_panel.push_back(list[t]);
    }
  }
  list_off[nreg] = (int32_t)list.size();
  const int64_t m = (int64_t)row_panel.size();
  if (m != cols) return ctx->fail(GBEM_ENUMERIC, "block system is not square");
  int rc = gbem_internal_ensure_matrix(ctx, m);
  if (rc) return rc;
  GBEM_CUDA(ctx, cudaMemsetAsync(ctx->d_A, 0, sizeof(double) * ctx->lda * m, ctx->stream));
  if (ctx->rhs_cap < (size_t)m) {
    cudaFree(ctx->d_rhs);
    ctx->d_rhs = nullptr;
    ctx->rhs_cap = 0;
    GBEM_CUDA(ctx, cudaMalloc(&ctx->d_rhs, 2 * (size_t)m * sizeof(double)));
    ctx->rhs_cap = m;
  }
  std::vector<int32_t> blob;
  auto put = [&](const std::vector<int32_t>& v) {
    size_t o = blob.size();
    blob.insert(blob.end(), v.begin(), v.end());
    return o;
  };
  const size_t o_rr = put(row_region), o_rp = put(row_panel), o_lo = put(list_off), o_l = put(list), o_id = put(ids);
  int32_t* d_blob = nullptr;
  double* d_eps = nullptr;
  BPanel* d_bp = nullptr;
  GBEM_CUDA(ctx, cudaMalloc(&d_blob, sizeof(int32_t) * blob.size()));
  GBEM_CUDA(ctx, cudaMalloc(&d_eps, sizeof(double) * nreg));
  GBEM_CUDA(ctx, cudaMalloc(&d_bp, sizeof(BPanel) * n));
  GBEM_CUDA(ctx, cudaMemcpy(d_blob, blob.data(), sizeof(int32_t) * blob.size(), cudaMemcpyHostToDevice));
  GBEM_CUDA(ctx, cudaMemcpy(d_eps, eps.data(), sizeof(double) * nreg, cudaMemcpyHostToDevice));
  GBEM_CUDA(ctx, cudaMemcpy(d_bp, bp.data(), sizeof(BPanel) * n, cudaMemcpyHostToDevice));
  unsigned long long* d_flags = nullptr;
  unsigned long long h_flags[2] = {0, 0};
  if (!galerkin) {
    k_collocation<<<(unsigned)((m * 32 + 255) / 256), 256, 0, ctx->stream>>>(
        d_bp, d_blob + o_rr, d_blob + o_rp, d_blob + o_lo, d_blob + o_l, d_blob + o_id, d_eps, nreg, (int)m, ctx->d_A,
        ctx->lda, ctx->d_rhs);
    GBEM_LAUNCH_CHECK(ctx);
  } else {
    if (m > 65535) return ctx->fail(GBEM_EINVAL, "Galerkin block system limited to 65535 rows");
    double rel_tol = cfg && cfg->rel_tol > 0 ? cfg->rel_tol : 1e-8;
    int levels = cfg && cfg->max_levels > 0 ? cfg->max_levels : 16;
    if (levels > kRombMax) return ctx->fail(GBEM_EINVAL, "max_levels exceeds 20");
    int lmax = 0;
    for (int k = 0; k < nreg; ++k) lmax = std::max(lmax, list_off[k + 1] - list_off[k]);
    GBEM_CUDA(ctx, cudaMalloc(&d_flags, sizeof(h_flags)));
    GBEM_CUDA(ctx, cudaMemsetAsync(d_flags, 0, sizeof(h_flags), ctx->stream));
    GBEM_CUDA(ctx, cudaMemsetAsync(ctx->d_rhs, 0, sizeof(double) * m, ctx->stream));
    k_galerkin_multi<<<dim3((unsigned)((lmax + 3) / 4), (unsigned)m), 128, 0, ctx->stream>>>(
        d_bp, d_blob + o_rr, d_blob + o_rp, d_blob + o_lo, d_blob + o_l, d_blob + o_id, d_eps, nreg, ctx->d_A,
        ctx->lda, ctx->d_rhs, rel_tol, levels, d_flags);
    GBEM_LAUNCH_CHECK(ctx);
    GBEM_CUDA(ctx, cudaMemcpyAsync(h_flags, d_flags, sizeof(h_flags), cudaMemcpyDeviceToHost, ctx->stream));
  }
  GBEM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  cudaFree(d_blob);
  cudaFree(d_eps);
  cudaFree(d_bp);
  if (d_flags) cudaFree(d_flags);
  if (h_flags[1]) return ctx->fail(GBEM_ENUMERIC, "non-finite integrand sample in the Galerkin block system");
  if (m_out) *m_out = m;
  if (nonconv_out) *nonconv_out = (int64_t)h_flags[0];
  return GBEM_OK;
}

int gbem_internal_assemble_collocation(gbem_ctx* ctx, const gbem_block_panels* P, int64_t n,
                                       const gbem_region* regions, int32_t nreg, int32_t main_net, int64_t* m_out) {
  return gbem_internal_assemble_block(ctx, P, n, regions, nreg, main_net, false, nullptr, m_out, nullptr);
}

// lu_solve (solver.hpp:53-88) of the context matrix with right-hand side
// d_b (device, length m, overwritten by the permuted system); x and the
// relative residual on the device.
int gbem_internal_lu_solve(gbem_ctx* ctx, double* d_b, double* d_x, double* d_resid, gbem_solve_stats* stats) {
  const int m = (int)ctx->n;
  const long long lda = ctx->lda;
  cudaStream_t s = ctx->stream;
  if (stats) {
    *stats = gbem_solve_stats{};
    stats->n = m;
    stats->nrhs = 1;
    stats->bad_pivot = -1;
  }
  if (m == 0) return GBEM_OK;
  // copies of A and b for the residual, pivots, scratch
  const size_t need = (size_t)lda * m + 4 * (size_t)m + 2 * 1024;
  if (ctx->work_cap < need) {
    cudaFree(ctx->d_work);
    ctx->d_work = nullptr;
    ctx->work_cap = 0;
    GBEM_CUDA(ctx, cudaMalloc(&ctx->d_work, need * sizeof(double)));
    ctx->work_cap = need;
  }
  double* A0 = ctx->d_work;
  double* b0 = A0 + (size_t)lda * m;
  double* rv = b0 + m;
  double* zv = rv + m;
  int* piv = reinterpret_cast<int*>(zv + m);
  double* part = zv + 2 * m;
  if (!ctx->d_info) {
    GBEM_CUDA(ctx, cudaMalloc(&ctx->d_info, sizeof(int)));
    GBEM_CUDA(ctx, cudaMallocHost(&ctx->h_info, sizeof(int)));
  }
  unsigned long long* d_max = reinterpret_cast<unsigned long long*>(part + 2 * 1000);
  cudaEvent_t e0 = ctx->ev[0], e1 = ctx->ev[1], e2 = ctx->ev[2];
  cudaEventRecord(e0, s);
  GBEM_CUDA(ctx, cudaMemcpyAsync(A0, ctx->d_A, sizeof(double) * lda * m, cudaMemcpyDeviceToDevice, s));
  GBEM_CUDA(ctx, cudaMemcpyAsync(b0, d_b, sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
  GBEM_CUDA(ctx, cudaMemsetAsync(d_max, 0, sizeof(unsigned long long), s));
  k_absmax<<<ctx->num_sms * 4, 256, 0, s>>>(ctx->d_A, lda, m, d_max);
  GBEM_LAUNCH_CHECK(ctx);
  unsigned long long hmax = 0;
  GBEM_CUDA(ctx, cudaMemcpyAsync(&hmax, d_max, sizeof(hmax), cudaMemcpyDeviceToHost, s));
  int big = 0x7fffffff;
  GBEM_CUDA(ctx, cudaMemcpyAsync(ctx->d_info, &big, sizeof(int), cudaMemcpyHostToDevice, s));
  GBEM_CUDA(ctx, cudaStreamSynchronize(s));
  double scale;
  memcpy(&scale, &hmax, sizeof(double));
  double thresh = 1e-14 * scale;
  if (!(ctx->attr_set & gbem_ctx::kAttrGemmLU)) {
    GBEM_CUDA(ctx, cudaFuncSetAttribute(gbem_gemm::k_gemm_g<gbem_gemm::kSub, 1>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gbem_gemm::kGSmem));
    ctx->attr_set |= gbem_ctx::kAttrGemmLU;
  }
  double* A = ctx->d_A;
  int grid = ctx->num_sms;
  if (grid > 1000) grid = 1000;
  for (int k0 = 0; k0 < m; k0 += LNB) {
    int nb = std::min(LNB, m - k0);
    int mm = m, kk0 = k0, nbb = nb;
    void* args[] = {(void*)&A, (void*)&lda, (void*)&mm, (void*)&kk0, (void*)&nbb, (void*)&d_b, (void*)&piv,
                    (void*)&thresh, (void*)&part, (void*)&ctx->d_info};
    GBEM_CUDA(ctx, cudaLaunchCooperativeKernel((void*)k_lu_panel, dim3(grid), dim3(kLuThreads), args, 0, s));
    GBEM_LAUNCH_CHECK(ctx);
    const int rest = m - k0 - nb;
    if (rest <= 0) continue;
    k_lu_trsm<<<(unsigned)((rest + 127) / 128), 128, 0, s>>>(A, lda, m, k0, nb);
    GBEM_LAUNCH_CHECK(ctx);
    const int vec = lda % 2 == 0 ? 1 : 0;
    gbem_gemm::k_gemm_g<gbem_gemm::kSub, 1><<<dim3((rest + 63) / 64, (rest + 63) / 64), gbem_gemm::kGThreads,
                                              gbem_gemm::kGSmem, s>>>(
        A + (long long)(k0 + nb) * lda + k0 + nb, lda, A + (long long)k0 * lda + k0 + nb, lda,
        A + (long long)(k0 + nb) * lda + k0, lda, rest, rest, nb, vec);
    GBEM_LAUNCH_CHECK(ctx);
  }
  cudaEventRecord(e1, s);
  GBEM_CUDA(ctx, cudaMemcpyAsync(ctx->h_info, ctx->d_info, sizeof(int), cudaMemcpyDeviceToHost, s));
  GBEM_CUDA(ctx, cudaStreamSynchronize(s));
  ctx->factored = true;
  if (*ctx->h_info != big) {
    if (stats) stats->bad_pivot = *ctx->h_info;
    return ctx->fail(GBEM_ENUMERIC, "matrix numerically singular (smallest pivot at row " +
                                        std::to_string(*ctx->h_info) + ")");
  }
  {
    int mm = m;
    void* args[] = {(void*)&A, (void*)&lda, (void*)&mm, (void*)&d_b, (void*)&zv, (void*)&d_x};
    GBEM_CUDA(ctx, cudaLaunchCooperativeKernel((void*)k_lu_solve, dim3(grid), dim3(kLuThreads), args, 0, s));
    GBEM_LAUNCH_CHECK(ctx);
  }
  cudaEventRecord(e2, s);
  k_gemv_resid<<<(unsigned)((m + 127) / 128), 128, 0, s>>>(A0, lda, m, d_x, b0, rv);
  GBEM_LAUNCH_CHECK(ctx);
  if (d_resid) {
    k_norm_ratio<<<1, 256, 0, s>>>(rv, b0, m, d_resid);
    GBEM_LAUNCH_CHECK(ctx);
  }
  GBEM_CUDA(ctx, cudaStreamSynchronize(s));
  if (stats) {
    float a = 0, c = 0;
    cudaEventElapsedTime(&a, e0, e1);
    cudaEventElapsedTime(&c, e1, e2);
    stats->ms_factor = a;
    stats->ms_solve = c;
    if (d_resid) GBEM_CUDA(ctx, cudaMemcpy(&stats->max_residual, d_resid, sizeof(double), cudaMemcpyDeviceToHost));
  }
  return GBEM_OK;
}

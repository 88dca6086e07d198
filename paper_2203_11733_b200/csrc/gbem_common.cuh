// gbem_common.cuh — shared device definitions for the B200 GBEM kernels.
//
// Panel geometry follows the reference Rect (proj/include/gbem/geometry.hpp:52-76):
// a rectangle in the plane x[axis] == level with spans a=[a0,a1], b=[b0,b1]
// along the two in-plane axes in axis-index order (inplaneAxes, geometry.hpp:41-47).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <math_constants.h>

namespace gbem_gpu {

// 48-byte panel record: three 16-byte vector loads per panel.
struct __align__(16) DPanel {
  double level, a0, a1, b0, b1;
  int axis;
  int pad;
};

constexpr double kFourPi = 4.0 * 3.14159265358979323846;  // oracle.hpp:11
constexpr int kQMax = 8;                                   // max far-field Gauss order per direction

// Pair classes (queue key < kFarKeyBase); far keys above (far_key).
enum PairClass : uint32_t {
  kClsCoplanar = 1,   // coplanar closed form (self, touching, near coplanar): kernels.hpp:86-94
  // offset-parallel / orthogonal near pairs on the reference's reduced 1-D
  // integrands (kernels.hpp:138-153, 175-214) with graded Gauss-Legendre,
  // band b = 0..3 -> 20 / 24 / 32 / 48 nodes per half segment
  kClsParallelGL = 2,    // keys 2..5
  kClsOrthogonalGL = 6,  // keys 6..9
  // near-contact pairs (gap < 1e-3 diameters, not touching): the reference's
  // adaptive Romberg (quadrature.hpp:27-113), one warp per pair
  kClsParallel = 10,
  kClsOrthogonal = 11,
  kFarKeyBase = 16,
};
constexpr int kNumKeys = 1 << 16;

// Far keys hold the three per-axis node-list sizes of the difference-set rule
// (gbem_assembly.cu, far_plan_code), sorted descending: m1 (the inner, register-
// resident list, <= 24) is the most significant field, so the queue segment
// of one m1 is contiguous and runs in its own kernel k_far<m1>; pairs with
// equal (m1, m2, m3) are contiguous, so a warp's loops are uniform.
//   key = kFarKeyBase + ((m1-1) << 8 | (m2-1) << 3 | (m3-1)),  m2 <= 24, m3 <= 8
constexpr int kFarListMax = 24;
__host__ __device__ inline uint32_t far_key(int m1, int m2, int m3) {
  return 16u + (uint32_t)(((m1 - 1) << 8) | ((m2 - 1) << 3) | (m3 - 1));
}
__host__ __device__ inline uint32_t far_key_first(int m1) { return 16u + (uint32_t)((m1 - 1) << 8); }

// Specialised far keys (gbem_assembly.cu, k_far_orth / k_far_par): pairs whose
// inner list has one of the kFastDescs descriptors (index d) run in a kernel
// compiled for that descriptor, the other two lists generated inside the node
// loops.  Orthogonal pairs (inner = the shared axis; two single rules of
// orders m2 >= m3):   key = kFastOrthBase + (d << 6 | (m2-1) << 3 | (m3-1))
// Parallel pairs (middle = the other shared axis with descriptor
// c2 = tent | (q1-1) << 1 | q2 << 4; the normal offset is a constant):
//                     key = kFastParBase + (d << 8 | c2)
constexpr uint32_t kFastOrthBase = 8192, kFastParBase = 16384;
constexpr int kFastMax = 32;  // descriptor indices d < kFastMax

// Queue entry: i (24 bits) | j (24 bits) | key (16 bits).
__host__ __device__ inline uint64_t pack_entry(uint32_t i, uint32_t j, uint32_t key) {
  return ((uint64_t)i << 40) | ((uint64_t)j << 16) | (uint64_t)key;
}
__host__ __device__ inline uint32_t entry_i(uint64_t e) { return (uint32_t)(e >> 40); }
__host__ __device__ inline uint32_t entry_j(uint64_t e) { return (uint32_t)((e >> 16) & 0xFFFFFFu); }
__host__ __device__ inline uint32_t entry_key(uint64_t e) { return (uint32_t)(e & 0xFFFFu); }

// In-plane axes ordered by axis index (geometry.hpp:41-47).
__host__ __device__ inline int ip0(int axis) { return axis == 0 ? 1 : 0; }
__host__ __device__ inline int ip1(int axis) { return axis == 2 ? 1 : 2; }

// World extent of a panel along axis k (Rect::extent, geometry.hpp:62-66).
__host__ __device__ inline void panel_extent(const DPanel& p, int k, double& lo, double& hi) {
  if (k == p.axis) {
    lo = p.level;
    hi = p.level;
  } else if (k == ip0(p.axis)) {
    lo = p.a0;
    hi = p.a1;
  } else {
    lo = p.b0;
    hi = p.b1;
  }
}

// rectDistance (geometry.hpp:79-87): gap between closed world extents.
__host__ __device__ inline double panel_gap(const DPanel& a, const DPanel& b) {
  double s = 0.0;
  for (int k = 0; k < 3; ++k) {
    double la, ha, lb, hb;
    panel_extent(a, k, la, ha);
    panel_extent(b, k, lb, hb);
    double g = fmax(fmax(lb - ha, la - hb), 0.0);
    s += g * g;
  }
  return sqrt(s);
}

__device__ __forceinline__ DPanel load_panel(const DPanel* __restrict__ P, uint32_t i) {
  const double2* q = reinterpret_cast<const double2*>(P + i);
  double2 x = __ldg(q), y = __ldg(q + 1), z = __ldg(q + 2);
  DPanel p;
  p.level = x.x;
  p.a0 = x.y;
  p.a1 = y.x;
  p.b0 = y.y;
  p.b1 = z.x;
  p.axis = __double_as_longlong(z.y) & 0xFF;
  p.pad = 0;
  return p;
}

// FP64 reciprocal square root: MUFU.RSQ64H seed + one third-order Householder
// step (max rel. error 2.7e-16 measured on B200, tools/fp64_peaks.cu).
// 5 FP64-pipe instructions; the argument is a strictly positive squared distance.
__device__ __forceinline__ double rsq64(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x * y, y, 1.0);
  return fma(y * e, fma(0.375, e, 0.5), y);
}

}  // namespace gbem_gpu

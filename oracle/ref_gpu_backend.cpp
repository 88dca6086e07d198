// ref_gpu_backend.cpp — TEST INFRASTRUCTURE: the reference-side binding of
// INTEGRATION.md §1 compiled against the UNMODIFIED reference headers
// (-I/root/reference/proj/include) and linked to this repository's
// libgbem_gpu.so, so the drop-in boundary is exercised exactly as a maintainer
// would bind it from capacitance_row (extraction.hpp:125-130).
//
// Only the Eigen-free reference headers are usable here (Eigen is absent), so
// gbem::GpuBackend returns the solution as a std::vector instead of the
// reference's Eigen-typed Solution; everything else is INTEGRATION.md's code.
// The scene, the per-main-net partition (partition_scene, partition.hpp:214)
// and the QuadratureConfig are the reference's own types; the charge reduction
// restates net_charges (extraction.hpp:55-79) for the all-Dirichlet single
// path.  Output: oracle/_ref/libgbem_ref_gpu.so (tests/test_gpu_extract.py).
#include <cstdint>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "gbem/errors.hpp"
#include "gbem/partition.hpp"
#include "gbem/quadrature.hpp"
#include "gbem_gpu.h"

namespace gbem {

struct GpuBackend {
  gbem_ctx* ctx = nullptr;
  explicit GpuBackend(int device = 0) {
    if (gbem_ctx_create(device, &ctx) != GBEM_OK)
      throw NumericalError(std::string("GPU: ") + (ctx ? gbem_last_error(ctx) : "no context"));
  }
  ~GpuBackend() { gbem_ctx_destroy(ctx); }
  GpuBackend(const GpuBackend&) = delete;
  GpuBackend& operator=(const GpuBackend&) = delete;

  static void check(gbem_ctx* c, int rc) {
    if (rc == GBEM_EINVAL) throw ValidationError(gbem_last_error(c));
    if (rc != GBEM_OK) throw NumericalError(gbem_last_error(c));
  }

  // replaces assemble_single (assembly.hpp:82) + cholesky_solve (solver.hpp:24)
  std::vector<double> solve_single(const PanelSet& ps, const QuadratureConfig& cfg, double* residual,
                                   bool* allConverged) {
    const size_t n = ps.panels.size();
    std::vector<uint8_t> ax(n);
    std::vector<double> lv(n), a0(n), a1(n), b0(n), b1(n), b(n), x(n);
    for (size_t k = 0; k < n; ++k) {
      const Rect& r = ps.panels[k].rect;
      ax[k] = (uint8_t)r.axis;
      lv[k] = r.level;
      a0[k] = r.spanA.lo;
      a1[k] = r.spanA.hi;
      b0[k] = r.spanB.lo;
      b1[k] = r.spanB.hi;
      b[k] = ps.panels[k].kind == FaceKind::ConductorSurface && ps.panels[k].netId == ps.mainNetId;
    }
    gbem_panels P{ax.data(), lv.data(), a0.data(), a1.data(), b0.data(), b1.data()};
    gbem_quad_config q{cfg.relTol, cfg.maxLevels, 0.0, 0.0};
    gbem_assembly_stats as{};
    gbem_solve_stats ss{};
    double resid = 0;
    check(ctx, gbem_assemble_single(ctx, &P, (int64_t)n, &q, nullptr, 0, &as));
    check(ctx, gbem_spd_solve(ctx, b.data(), 1, x.data(), &resid, &ss));
    if (allConverged) *allConverged = as.not_converged == 0;
    if (residual) *residual = resid;
    return x;
  }
};

}  // namespace gbem

namespace {

gbem::Scene build(const double* dom, int nreg, const double* regs, int ncell, const double* cells, const int* bc) {
  gbem::Cuboid domain{{dom[0], dom[1], dom[2]}, {dom[3], dom[4], dom[5]}};
  std::vector<gbem::DielectricRegion> regions;
  for (int r = 0; r < nreg; ++r) {
    const double* q = regs + 8 * r;
    regions.push_back({static_cast<int>(q[0]), gbem::Cuboid{{q[2], q[3], q[4]}, {q[5], q[6], q[7]}}, q[1]});
  }
  std::vector<gbem::Conductor> conductors;
  for (int c = 0; c < ncell; ++c) {
    const double* q = cells + 7 * c;
    int id = static_cast<int>(q[0]);
    gbem::Cuboid cub{{q[1], q[2], q[3]}, {q[4], q[5], q[6]}};
    bool found = false;
    for (auto& cd : conductors)
      if (cd.netId == id) {
        cd.cuboids.push_back(cub);
        found = true;
      }
    if (!found) conductors.push_back(gbem::Conductor{id, {cub}});
  }
  std::array<gbem::OuterBC, 6> obc;
  for (int k = 0; k < 6; ++k) obc[k] = bc[k] ? gbem::OuterBC::Neumann : gbem::OuterBC::Dirichlet;
  return gbem::build_scene(domain, regions, conductors, obc);
}

}  // namespace

extern "C" {

// capacitance_row (extraction.hpp:106-160, single-dielectric all-Dirichlet
// branch) through gbem::GpuBackend: the reference's scene and partition, the
// B200 assembly + Cholesky.  charges[k] = charge of the k-th net in ascending
// net-id order (F); *outer = charge on the grounded outer panels; returns the
// net count, -1 ValidationError, -2 NumericalError (message in err).
int refgpu_capacitance_row(const double* dom, int nreg, const double* regs, int ncell, const double* cells,
                           const int* bc, const double* params, int main_net, double rel_tol, int max_levels,
                           double* charges, int cap, double* outer, int64_t* panels, double* residual,
                           int* converged, char* err, int errlen) {
  try {
    gbem::Scene s = build(dom, nreg, regs, ncell, cells, bc);
    gbem::PartitionParams pp;
    pp.p1 = params[0];
    pp.p2 = params[1];
    pp.p3 = params[2];
    pp.p5 = params[3];
    gbem::PanelSet ps = gbem::partition_scene(s, main_net, pp);
    if (s.regions.size() != 1) throw gbem::ValidationError("binding test: single-dielectric scenes only");
    gbem::QuadratureConfig q;
    q.relTol = rel_tol;
    q.maxLevels = max_levels;
    gbem::GpuBackend gpu(0);
    bool conv = true;
    double res = 0;
    std::vector<double> x = gpu.solve_single(ps, q, &res, &conv);
    // net_charges (extraction.hpp:55-79): Q = eps_r eps0 x kUnitScale summed per net
    const double kEps0 = 8.854187817e-12, kUnitScale = 1e-6;  // extraction.hpp:20-21
    std::map<int, double> Q;
    for (const auto& c : s.conductors) Q[c.netId] = 0.0;
    double out = 0.0;
    for (size_t k = 0; k < ps.panels.size(); ++k) {
      const gbem::Panel& p = ps.panels[k];
      if (p.kind == gbem::FaceKind::Interface || p.kind == gbem::FaceKind::NeumannOuter) continue;
      const gbem::DielectricRegion* reg = s.regionById(p.regionA);
      if (!reg) throw gbem::ValidationError("missing permittivity for region " + std::to_string(p.regionA));
      const double v = reg->relPermittivity * kEps0 * x[k] * kUnitScale;
      if (p.kind == gbem::FaceKind::ConductorSurface)
        Q[p.netId] += v;
      else
        out += v;
    }
    int i = 0;
    for (const auto& [id, v] : Q)
      if (i < cap) charges[i++] = v;
    if (outer) *outer = out;
    if (panels) *panels = (int64_t)ps.panels.size();
    if (residual) *residual = res;
    if (converged) *converged = conv ? 1 : 0;
    return (int)Q.size();
  } catch (const gbem::ValidationError& e) {
    if (err && errlen > 0) {
      std::strncpy(err, e.what(), errlen - 1);
      err[errlen - 1] = 0;
    }
    return -1;
  } catch (const std::exception& e) {
    if (err && errlen > 0) {
      std::strncpy(err, e.what(), errlen - 1);
      err[errlen - 1] = 0;
    }
    return -2;
  }
}

}  // extern "C"

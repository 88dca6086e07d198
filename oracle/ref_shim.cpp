// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" wrapper that compiles the UNMODIFIED reference headers in
// place (-I/root/reference/proj/include) into oracle/_ref/libgbem_ref.so.  No
// reference source is copied into this repo; only the Eigen-free headers are
// used (geometry, partition, quadrature, oracle, kernels).  The Eigen-dependent
// pieces (assemble_single, cholesky_solve) are restated in oracle/gbem_oracle.c.
//
// Consumers: tests/ (parity pins), bench.py --impl reference and the
// cpu_baseline leg.  The product never loads this library.
#include <atomic>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "gbem/kernels.hpp"
#include "gbem/oracle.hpp"
#include "gbem/partition.hpp"

#include "gbem_oracle.h"

namespace {

gbem::Rect toRect(const orc_rect& r) {
  gbem::Rect o;
  o.axis = r.axis;
  o.level = r.level;
  o.spanA = {r.a0, r.a1};
  o.spanB = {r.b0, r.b1};
  o.normalSign = 1;
  return o;
}

}  // namespace

extern "C" {

// gbem::u_point_rect / q_point_rect (kernels.hpp:319-355).
double ref_u_point_rect(const double x[3], const orc_rect* r) {
  return gbem::u_point_rect(gbem::Vec3{x[0], x[1], x[2]}, toRect(*r));
}
double ref_q_point_rect(const double x[3], const orc_rect* r, int nsign) {
  gbem::Rect R = toRect(*r);
  R.normalSign = nsign;
  return gbem::q_point_rect(gbem::Vec3{x[0], x[1], x[2]}, R);
}


// gbem::q_pair_integral (kernels.hpp:295): test a, source b with normal sign nsign.
orc_kv ref_q_pair_integral(const orc_rect* a, const orc_rect* b, int nsign, double rel_tol, int max_levels) {
  orc_kv out{0.0, 1, 0, 0};
  gbem::QuadratureConfig cfg;
  cfg.relTol = rel_tol;
  cfg.maxLevels = max_levels;
  gbem::Rect B = toRect(*b);
  B.normalSign = nsign;
  try {
    gbem::KernelValue kv = gbem::q_pair_integral(toRect(*a), B, cfg);
    out.value = kv.value;
    out.converged = kv.converged ? 1 : 0;
    out.evals = kv.evals;
  } catch (...) {
    out.status = 2;
  }
  return out;
}

// gbem::u_pair_integral (kernels.hpp:270) with a QuadratureConfig.
orc_kv ref_u_pair_integral(const orc_rect* a, const orc_rect* b, double rel_tol,
                           int max_levels) {
  orc_kv out{0.0, 1, 0, 0};
  gbem::QuadratureConfig cfg;
  cfg.relTol = rel_tol;
  cfg.maxLevels = max_levels;
  try {
    gbem::KernelValue kv = gbem::u_pair_integral(toRect(*a), toRect(*b), cfg);
    out.value = kv.value;
    out.converged = kv.converged ? 1 : 0;
    out.evals = kv.evals;
  } catch (const gbem::NumericalError&) {
    out.status = 2;
  }
  return out;
}

// Reference kernel over a pair list on nthreads host threads (SPEC.md:285
// permits evaluating independent pairs in parallel).
int ref_u_pairs(int64_t npairs, const orc_rect* a, const orc_rect* b, double rel_tol,
                int max_levels, double* out, int* converged, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  std::atomic<int> status{0};
  std::atomic<int64_t> next{0};
  const int64_t grain = 64;
  auto work = [&] {
    for (;;) {
      int64_t s = next.fetch_add(grain);
      if (s >= npairs) break;
      int64_t e = std::min(npairs, s + grain);
      for (int64_t k = s; k < e; ++k) {
        orc_kv kv = ref_u_pair_integral(&a[k], &b[k], rel_tol, max_levels);
        out[k] = kv.value;
        if (converged) converged[k] = kv.converged;
        if (kv.status) status = kv.status;
      }
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nthreads; ++t) th.emplace_back(work);
  work();
  for (auto& t : th) t.join();
  return status.load();
}

// The reference's assemble_single loop (assembly.hpp:88-102) around the
// reference kernel, rows dealt dynamically to nthreads threads.  A is n x n
// row-major, both triangles written.
int ref_assemble_single(int64_t n, const orc_rect* p, double rel_tol, int max_levels,
                        double* A, int* all_converged, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  std::atomic<int> status{0}, conv{1};
  std::atomic<int64_t> next{0};
  auto work = [&] {
    for (;;) {
      int64_t i = next.fetch_add(1);
      if (i >= n) break;
      gbem::Rect ri = toRect(p[i]);
      double ai = ri.area();
      for (int64_t j = i; j < n; ++j) {
        gbem::Rect rj = toRect(p[j]);
        gbem::QuadratureConfig cfg;
        cfg.relTol = rel_tol;
        cfg.maxLevels = max_levels;
        try {
          gbem::KernelValue kv = gbem::u_pair_integral(ri, rj, cfg);
          if (!kv.converged) conv = 0;
          double v = kv.value / (ai * rj.area());
          A[i * n + j] = v;
          A[j * n + i] = v;
        } catch (const gbem::NumericalError&) {
          status = 2;
        }
      }
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nthreads; ++t) th.emplace_back(work);
  work();
  for (auto& t : th) t.join();
  if (all_converged) *all_converged = conv.load();
  return status.load();
}

// ref_assemble_single plus the reference's convergence diagnostics: the
// (i, j) of every pair whose u_pair_integral reports converged = false
// (assembly.hpp:97 ANDs these flags into GalerkinSystem::converged), up to
// nc_cap of them; *nc_count receives the total.  Rows are dealt in chunks of
// `chunk` so a progress callback can report.
int ref_assemble_single_diag(int64_t n, const orc_rect* p, double rel_tol, int max_levels,
                             double* A, int64_t* nc_pairs, int64_t nc_cap, int64_t* nc_count,
                             int nthreads, void (*progress)(int64_t rows_done)) {
  if (nthreads < 1) nthreads = 1;
  std::atomic<int> status{0};
  std::atomic<int64_t> next{0}, nnc{0}, done{0};
  auto work = [&] {
    for (;;) {
      int64_t i = next.fetch_add(1);
      if (i >= n) break;
      gbem::Rect ri = toRect(p[i]);
      double ai = ri.area();
      for (int64_t j = i; j < n; ++j) {
        gbem::Rect rj = toRect(p[j]);
        gbem::QuadratureConfig cfg;
        cfg.relTol = rel_tol;
        cfg.maxLevels = max_levels;
        try {
          gbem::KernelValue kv = gbem::u_pair_integral(ri, rj, cfg);
          if (!kv.converged) {
            int64_t s = nnc.fetch_add(1);
            if (s < nc_cap) {
              nc_pairs[2 * s] = i;
              nc_pairs[2 * s + 1] = j;
            }
          }
          double v = kv.value / (ai * rj.area());
          A[i * n + j] = v;
          A[j * n + i] = v;
        } catch (const gbem::NumericalError&) {
          status = 2;
        }
      }
      int64_t d = done.fetch_add(1) + 1;
      if (progress && d % 256 == 0) progress(d);
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nthreads; ++t) th.emplace_back(work);
  work();
  for (auto& t : th) t.join();
  if (nc_count) *nc_count = nnc.load();
  return status.load();
}

// gbem::oracle_pair_integral(SingleLayer) (oracle.hpp:191).
double ref_oracle_pair_integral(const orc_rect* a, const orc_rect* b, int depth) {
  return gbem::oracle_pair_integral(gbem::KernelKind::SingleLayer, toRect(*a), toRect(*b),
                                    depth);
}

// gbem::oracle_pair_integral(DoubleLayer) (oracle.hpp:191, the Q branch).
double ref_q_oracle_pair_integral(const orc_rect* a, const orc_rect* b, int nsign, int depth) {
  gbem::Rect B = toRect(*b);
  B.normalSign = nsign;
  return gbem::oracle_pair_integral(gbem::KernelKind::DoubleLayer, toRect(*a), B, depth);
}

// gbem::rectDistance (geometry.hpp:79).
double ref_rect_distance(const orc_rect* a, const orc_rect* b) {
  return gbem::rectDistance(toRect(*a), toRect(*b));
}

// Scene -> gbem::build_scene (geometry.hpp:237) -> gbem::partition_scene
// (partition.hpp:214) for one main net.  Flat scene description:
//   dom[6] = lo xyz, hi xyz; regions: nreg x (id, eps, lo xyz, hi xyz) = 8 doubles;
//   cells: ncell x (netId, lo xyz, hi xyz) = 7 doubles; bc[6] (0 dirichlet, 1 neumann);
//   params[4] = p1 p2 p3 p5.
// Output panel arrays of capacity cap; returns the panel count (> cap means
// retry with a larger buffer), -1 on ValidationError (message in err).
// Per panel: ints[6] = axis, normalSign, kind, netId, regionA, regionB;
//            dbl[7]  = level, a0, a1, b0, b1, area, distToMain; facing[1].
int64_t ref_partition_scene(const double* dom, int nreg, const double* regs, int ncell,
                            const double* cells, const int* bc, const double* params,
                            int main_net, int64_t cap, int* ints, double* dbl, int* facing,
                            char* err, int errlen) {
  try {
    gbem::Cuboid domain{{dom[0], dom[1], dom[2]}, {dom[3], dom[4], dom[5]}};
    std::vector<gbem::DielectricRegion> regions;
    for (int r = 0; r < nreg; ++r) {
      const double* q = regs + 8 * r;
      regions.push_back({static_cast<int>(q[0]), gbem::Cuboid{{q[2], q[3], q[4]}, {q[5], q[6], q[7]}},
                         q[1]});
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
    for (int k = 0; k < 6; ++k)
      obc[k] = bc[k] ? gbem::OuterBC::Neumann : gbem::OuterBC::Dirichlet;
    gbem::Scene s = gbem::build_scene(domain, regions, conductors, obc);
    gbem::PartitionParams pp;
    pp.p1 = params[0];
    pp.p2 = params[1];
    pp.p3 = params[2];
    pp.p5 = params[3];
    gbem::PanelSet ps = gbem::partition_scene(s, main_net, pp);
    int64_t n = static_cast<int64_t>(ps.panels.size());
    if (n > cap) return n;
    for (int64_t i = 0; i < n; ++i) {
      const gbem::Panel& p = ps.panels[i];
      int* I = ints + 6 * i;
      double* D = dbl + 7 * i;
      I[0] = p.rect.axis;
      I[1] = p.rect.normalSign;
      I[2] = static_cast<int>(p.kind);
      I[3] = p.netId;
      I[4] = p.regionA;
      I[5] = p.regionB;
      D[0] = p.rect.level;
      D[1] = p.rect.spanA.lo;
      D[2] = p.rect.spanA.hi;
      D[3] = p.rect.spanB.lo;
      D[4] = p.rect.spanB.hi;
      D[5] = p.area;
      D[6] = p.distToMain;
      facing[i] = static_cast<int>(p.facing);
    }
    return n;
  } catch (const std::exception& e) {
    if (err && errlen > 0) {
      std::strncpy(err, e.what(), static_cast<size_t>(errlen - 1));
      err[errlen - 1] = 0;
    }
    return -1;
  }
}

}  // extern "C"

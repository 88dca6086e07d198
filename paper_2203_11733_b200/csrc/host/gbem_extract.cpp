// gbem_extract.cpp — capacitance extraction driver: the caller of the GPU
// boundary (include/gbem_gpu.h) in place of assemble_single + cholesky_solve
// (proj/include/gbem/extraction.hpp:106-184).
#include <chrono>
#include <cmath>
#include <cstring>

#include "../../../include/gbem_gpu.h"
#include "gbem_host.hpp"

namespace gbh {

namespace {

void raise(gbem_ctx* ctx, int rc) {
  if (rc == GBEM_OK) return;
  std::string msg = gbem_last_error(ctx);
  if (rc == GBEM_EINVAL) throw ValidationError(msg);
  if (rc == GBEM_ENUMERIC) throw NumericalError(msg);
  throw std::runtime_error("CUDA: " + msg);
}

struct SoA {
  std::vector<uint8_t> axis;
  std::vector<double> level, a0, a1, b0, b1;
  explicit SoA(const PanelSet& ps) {
    const size_t n = ps.panels.size();
    axis.resize(n);
    level.resize(n);
    a0.resize(n);
    a1.resize(n);
    b0.resize(n);
    b1.resize(n);
    for (size_t k = 0; k < n; ++k) {
      const Rect& r = ps.panels[k].r;
      axis[k] = (uint8_t)r.axis;
      level[k] = r.level;
      a0[k] = r.a.lo;
      a1[k] = r.a.hi;
      b0[k] = r.b.lo;
      b1[k] = r.b.hi;
    }
  }
  gbem_panels view() const { return {axis.data(), level.data(), a0.data(), a1.data(), b0.data(), b1.data()}; }
};

bool single_dielectric(const Scene& s) {
  if (s.regions.size() != 1) return false;
  if (s.freespace) return true;
  for (int b : s.bc)
    if (b != 0) return false;
  return true;
}

gbem_quad_config quad(const Options& o) {
  gbem_quad_config q{};
  q.rel_tol = o.rel_tol;
  q.max_levels = o.max_levels;
  return q;
}

}  // namespace

// The block (mixed-unknown) path of capacitance_row (extraction.hpp:132-143):
// GPU assemble_multi (the Galerkin block system, method "galerkin-block") or,
// for the collocation baseline, GPU assemble_collocation; then GPU lu_solve and
// net_charges through the flux-unknown columns (extraction.hpp:55-79).
static Row block_row(gbem_ctx* ctx, const Scene& s, const PanelSet& ps, int main_net, const Options& o) {
  const size_t n = ps.panels.size();
  Row row;
  row.main_net = main_net;
  row.diag.panels = n;
  row.diag.method = o.collocation ? "collocation" : "galerkin-block";
  SoA soa(ps);
  std::vector<int8_t> nsign(n);
  std::vector<int32_t> kind(n), net(n), ra(n), rb(n);
  for (size_t k = 0; k < n; ++k) {
    const Panel& pn = ps.panels[k];
    nsign[k] = (int8_t)pn.r.nsign;
    kind[k] = (int32_t)pn.kind;
    net[k] = pn.net;
    ra[k] = pn.regA;
    rb[k] = pn.regB;
  }
  gbem_block_panels bp{soa.view(), nsign.data(), kind.data(), net.data(), ra.data(), rb.data()};
  std::vector<gbem_region> regs;
  for (const Region& r : s.regions) regs.push_back(gbem_region{r.id, r.eps});
  auto t0 = std::chrono::steady_clock::now();
  int64_t m = 0;
  std::vector<double> A;
  const bool dump = !o.dump_matrix.empty();
  if (o.collocation) {
    raise(ctx, gbem_assemble_collocation(ctx, &bp, (int64_t)n, regs.data(), (int32_t)regs.size(), main_net, nullptr,
                                         0, nullptr, &m));
    if (dump) {
      A.resize((size_t)m * m);
      raise(ctx, gbem_assemble_collocation(ctx, &bp, (int64_t)n, regs.data(), (int32_t)regs.size(), main_net,
                                           A.data(), m, nullptr, &m));
    }
  } else {
    gbem_quad_config q{};
    q.rel_tol = o.rel_tol;
    q.max_levels = o.max_levels;
    int64_t mmax = (int64_t)n;
    for (size_t k = 0; k < n; ++k) mmax += ps.panels[k].kind == kInterface ? 1 : 0;
    if (dump) A.resize((size_t)mmax * mmax);
    int32_t conv = 1;
    raise(ctx, gbem_assemble_multi(ctx, &bp, (int64_t)n, regs.data(), (int32_t)regs.size(), main_net, &q,
                                   dump ? A.data() : nullptr, mmax, nullptr, &m, &conv));
    row.diag.converged = conv != 0;
    if (dump) {  // compact the mmax-strided copy to m x m
      for (int64_t r = 0; r < m; ++r)
        for (int64_t c = 0; c < m; ++c) A[(size_t)r * m + c] = A[(size_t)r * mmax + c];
      A.resize((size_t)m * m);
    }
  }
  if (dump) dump_matrix_file(o.dump_matrix, A, (size_t)m);  // dump_system_matrix (extraction.hpp:83-99)
  std::vector<double> x((size_t)m, 0.0);
  double resid = 0;
  gbem_solve_stats sst{};
  raise(ctx, gbem_lu_solve(ctx, nullptr, x.data(), &resid, &sst));
  auto t1 = std::chrono::steady_clock::now();
  row.diag.seconds = std::chrono::duration<double>(t1 - t0).count();
  row.diag.residual = resid;
  // qCol of buildUnknownMap (assembly.hpp:51-75)
  const size_t o3 = ps.offset[3];
  for (const Net& nn : s.nets) row.cap[nn.id] = 0.0;
  double outer = 0;
  for (size_t k = 0; k < n; ++k) {
    const Panel& pn = ps.panels[k];
    if (pn.kind == kInterface || pn.kind == kNeumann) continue;
    const size_t col = k;  // conductor / Dirichlet panels precede o3: qCol = index
    (void)o3;
    const Region* reg = s.region(pn.regA);
    if (!reg) throw ValidationError("missing permittivity for region " + std::to_string(pn.regA));
    const double qv = reg->eps * kEps0 * x[col] * kUnitScale;
    if (pn.kind == kConductor)
      row.cap[pn.net] += qv;
    else
      outer += qv;
  }
  row.outer = outer;
  bool all_dirichlet = s.freespace;
  if (!s.freespace) {
    all_dirichlet = true;
    for (int b : s.bc)
      if (b != 0) all_dirichlet = false;
  }
  if (all_dirichlet) {  // neutrality only for all-Dirichlet scenes (extraction.hpp:153-158)
    double total = outer;
    for (const auto& kv : row.cap) total += kv.second;
    row.diag.neutrality = std::abs(total) / std::max(std::abs(row.cap.at(main_net)), 1e-300);
  }
  return row;
}

Row capacitance_row(gbem_ctx* ctx, const Scene& s, int main_net, const Params& p, const Options& o) {
  PanelSet ps = partition_for_net(s, main_net, p);
  // single path iff one region, all-Dirichlet boundary and no collocation baseline (extraction.hpp:110-114)
  if (o.collocation || !single_dielectric(s)) return block_row(ctx, s, ps, main_net, o);
  if (ps.count(kNeumann) || ps.count(kInterface))
    throw ValidationError("single-dielectric assembly requires one region with an all-Dirichlet boundary");
  const size_t n = ps.panels.size();
  Row row;
  row.main_net = main_net;
  row.diag.panels = n;
  row.diag.method = "galerkin-single";
  SoA soa(ps);
  gbem_panels view = soa.view();
  gbem_quad_config q = quad(o);
  gbem_assembly_stats ast{};
  auto t0 = std::chrono::steady_clock::now();
  raise(ctx, gbem_assemble_single(ctx, &view, (int64_t)n, &q, nullptr, 0, &ast));
  row.diag.converged = ast.not_converged == 0;
  if (!o.dump_matrix.empty()) {
    std::vector<double> A(n * n);
    raise(ctx, gbem_matrix_download(ctx, A.data(), (int64_t)n));
    dump_matrix_file(o.dump_matrix, A, n);
  }
  // knownPotential (assembly.hpp:42-44): 1 on the main net's conductor panels
  std::vector<double> b(n, 0.0), x(n, 0.0);
  for (size_t k = 0; k < n; ++k)
    if (ps.panels[k].kind == kConductor && ps.panels[k].net == main_net) b[k] = 1.0;
  double resid = 0;
  gbem_solve_stats sst{};
  raise(ctx, gbem_spd_solve(ctx, b.data(), 1, x.data(), &resid, &sst));
  auto t1 = std::chrono::steady_clock::now();
  row.diag.seconds = std::chrono::duration<double>(t1 - t0).count();
  row.diag.residual = resid;
  // net_charges (extraction.hpp:55-79)
  for (const Net& nn : s.nets) row.cap[nn.id] = 0.0;
  double outer = 0;
  for (size_t k = 0; k < n; ++k) {
    const Panel& pn = ps.panels[k];
    const Region* reg = s.region(pn.regA);
    if (!reg) throw ValidationError("missing permittivity for region " + std::to_string(pn.regA));
    const double qv = reg->eps * kEps0 * x[k] * kUnitScale;
    if (pn.kind == kConductor)
      row.cap[pn.net] += qv;
    else
      outer += qv;
  }
  row.outer = outer;
  double total = outer;
  for (const auto& kv : row.cap) total += kv.second;
  row.diag.neutrality = std::abs(total) / std::max(std::abs(row.cap.at(main_net)), 1e-300);
  return row;
}

static void reciprocity(CapMatrix& cm) {
  cm.reciprocity = 0;
  for (size_t a = 0; a < cm.rows.size(); ++a)
    for (size_t b = a + 1; b < cm.rows.size(); ++b) {
      double cab = cm.rows[a].cap.at(cm.ids[b]), cba = cm.rows[b].cap.at(cm.ids[a]);
      double den = std::max(std::abs(cab), std::abs(cba));
      if (den > 0) cm.reciprocity = std::max(cm.reciprocity, std::abs(cab - cba) / den);
    }
}

CapMatrix capacitance_matrix(gbem_ctx* ctx, const Scene& s, const Params& p, const Options& o) {
  CapMatrix cm;
  for (const Net& n : s.nets) cm.ids.push_back(n.id);
  for (int id : cm.ids) {
    Options ro = o;
    if (!o.dump_matrix.empty()) ro.dump_matrix = o.dump_matrix + "_net" + std::to_string(id);
    cm.rows.push_back(capacitance_row(ctx, s, id, p, ro));
  }
  reciprocity(cm);
  return cm;
}

CapMatrix capacitance_matrix_shared(gbem_ctx* ctx, const Scene& s, const PanelSet& ps, const Options& o) {
  if (!single_dielectric(s))
    throw ValidationError("the GPU path solves the single-dielectric all-Dirichlet system");
  const size_t n = ps.panels.size();
  const size_t K = s.nets.size();
  if (K == 0) throw ValidationError("scene has no conductors");
  if (K > 8192) throw ValidationError("at most 8192 nets per shared solve");
  std::map<int, size_t> col;
  for (size_t k = 0; k < K; ++k) col[s.nets[k].id] = k;
  SoA soa(ps);
  gbem_panels view = soa.view();
  gbem_quad_config q = quad(o);
  gbem_assembly_stats ast{};
  std::vector<double> X, res(K, 0.0), Cpcg, outer_pcg;
  const bool pcg = o.solver == 2 || (o.solver == 0 && gbem_ctx_nranks(ctx) > 1);
  auto t0 = std::chrono::steady_clock::now();
  if (pcg) {
    // row-block sharded block-Jacobi PCG (gbem_pcg_extract_cmatrix; every rank
    // runs this with the same panels, the context's collectives join them)
    if (!o.dump_matrix.empty()) throw ValidationError("--dump-matrix needs the direct solver");
    std::vector<int32_t> net(n, -1);
    for (size_t p = 0; p < n; ++p)
      if (ps.panels[p].kind == kConductor) net[p] = (int32_t)col.at(ps.panels[p].net);
    const Region* reg = s.region(ps.panels.empty() ? 0 : ps.panels.front().regA);
    if (!reg) throw ValidationError("missing permittivity");
    gbem_pcg_options po{o.pcg_tol, 5000, std::max(1, o.jacobi_blocks)};
    gbem_pcg_stats pst{};
    Cpcg.assign(K * K, 0.0);
    outer_pcg.assign(K, 0.0);
    raise(ctx, gbem_pcg_extract_cmatrix(ctx, &view, (int64_t)n, net.data(), (int32_t)K, reg->eps, &q, &po,
                                        Cpcg.data(), res.data(), outer_pcg.data(), &ast, &pst));
  } else {
    raise(ctx, gbem_assemble_single(ctx, &view, (int64_t)n, &q, nullptr, 0, &ast));
    if (!o.dump_matrix.empty()) {
      std::vector<double> A(n * n);
      raise(ctx, gbem_matrix_download(ctx, A.data(), (int64_t)n));
      dump_matrix_file(o.dump_matrix, A, n);
    }
    std::vector<double> B(n * K, 0.0);
    X.assign(n * K, 0.0);
    for (size_t p = 0; p < n; ++p)
      if (ps.panels[p].kind == kConductor) B[col.at(ps.panels[p].net) * n + p] = 1.0;
    gbem_solve_stats sst{};
    raise(ctx, gbem_spd_solve(ctx, B.data(), (int64_t)K, X.data(), res.data(), &sst));
  }
  auto t1 = std::chrono::steady_clock::now();
  const double secs = std::chrono::duration<double>(t1 - t0).count();
  CapMatrix cm;
  for (const Net& nn : s.nets) cm.ids.push_back(nn.id);
  for (size_t r = 0; r < K; ++r) {
    Row row;
    row.main_net = s.nets[r].id;
    row.diag.panels = n;
    row.diag.method = pcg ? "galerkin-shared-pcg" : "galerkin-shared";
    row.diag.seconds = secs;
    row.diag.residual = res[r];
    row.diag.converged = ast.not_converged == 0;
    for (const Net& nn : s.nets) row.cap[nn.id] = 0.0;
    double outer = 0;
    if (pcg) {
      for (size_t k = 0; k < K; ++k) row.cap[s.nets[k].id] = Cpcg[r * K + k];
      outer = outer_pcg[r];
    } else {
      for (size_t p = 0; p < n; ++p) {
        const Panel& pn = ps.panels[p];
        const Region* reg = s.region(pn.regA);
        if (!reg) throw ValidationError("missing permittivity for region " + std::to_string(pn.regA));
        const double qv = reg->eps * kEps0 * X[r * n + p] * kUnitScale;
        if (pn.kind == kConductor)
          row.cap[pn.net] += qv;
        else
          outer += qv;
      }
    }
    row.outer = outer;
    double total = outer;
    for (const auto& kv : row.cap) total += kv.second;
    row.diag.neutrality = s.freespace ? -1.0 : std::abs(total) / std::max(std::abs(row.cap.at(row.main_net)), 1e-300);
    cm.rows.push_back(row);
  }
  reciprocity(cm);
  return cm;
}

}  // namespace gbh

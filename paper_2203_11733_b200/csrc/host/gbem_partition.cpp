// gbem_partition.cpp — a-priori graded panel partition.
//
// partition_for_net reproduces the reference scheme panel for panel, in the
// same order and with the same floating-point operations
// (proj/include/gbem/partition.hpp:60-245): per face a core strip over the
// main net's bounding-box footprint, then rings whose width doubles, each strip
// gridded uniformly against the area bound at its nearest distance.  The panel
// order defines the matrix row order, so the GPU system is the reference's
// system entry for entry.
//
// partition_uniform / partition_graded are the net-independent panelisations
// used by the BASELINE configs (one matrix, one right-hand side per net).
#include <algorithm>
#include <cmath>
#include <functional>

#include "gbem_host.hpp"

namespace gbh {

void Params::check() const {
  if (!(p1 > 0) || !(p2 >= 1) || !(p3 > 0) || !(p5 > 0) || !(exp_dirichlet > 0) || !(exp_soft > 0) ||
      !(aspect > 0))
    throw ValidationError("partition params must be strictly positive with p2 >= 1");
}

namespace {

Box bounding_box(const Net& n) {
  Box bb = n.cells.front();
  for (const Box& c : n.cells)
    for (int k = 0; k < 3; ++k) {
      bb.lo[k] = std::min(bb.lo[k], c.lo[k]);
      bb.hi[k] = std::max(bb.hi[k], c.hi[k]);
    }
  return bb;
}

// gridStrip (partition.hpp:92-134)
void grid_strip(const Rect& proto, Span sa, Span sb, double amax, double aspect, std::vector<Rect>& out) {
  const double wa = sa.len(), wb = sb.len();
  if (!(wa > 0.0) || !(wb > 0.0)) return;
  const double cell = std::sqrt(amax);
  auto first_count = [cell](double w) {
    double c = std::ceil(w / cell - 1e-12);
    return std::max<long long>(1, (long long)c);
  };
  long long na = first_count(wa), nb = first_count(wb);
  const double slack = 1.0 + 1e-12;
  auto ca = [&] { return wa / (double)na; };
  auto cb = [&] { return wb / (double)nb; };
  auto limit = [&] {
    if (na > 2000000 || nb > 2000000 || na * nb > 8000000)
      throw ValidationError("partition bound too small: cell limit exceeded");
  };
  limit();
  while (ca() * cb() > amax * slack) {
    (ca() >= cb() ? na : nb) += 1;
    limit();
  }
  while (std::max(ca(), cb()) > aspect * std::min(ca(), cb()) * slack) {
    (ca() >= cb() ? na : nb) += 1;
    limit();
  }
  for (long long ia = 0; ia < na; ++ia) {
    const double a0 = sa.lo + wa * (double)ia / (double)na;
    const double a1 = ia + 1 == na ? sa.hi : sa.lo + wa * (double)(ia + 1) / (double)na;
    for (long long ib = 0; ib < nb; ++ib) {
      const double b0 = sb.lo + wb * (double)ib / (double)nb;
      const double b1 = ib + 1 == nb ? sb.hi : sb.lo + wb * (double)(ib + 1) / (double)nb;
      Rect c = proto;
      c.a = Span{a0, a1};
      c.b = Span{b0, b1};
      out.push_back(c);
    }
  }
}

// clampSpan (partition.hpp:136-140)
Span clamp_to(Span s, Span lim) {
  double lo = std::min(std::max(s.lo, lim.lo), lim.hi);
  double hi = std::max(std::min(s.hi, lim.hi), lim.lo);
  return {std::min(lo, hi), std::max(lo, hi)};
}

// expandSpan (partition.hpp:144-149): grow by delta, snapping to the face rim
// when the leftover border would be thinner than the step.
Span grow_to(Span cur, Span lim, double delta) {
  double lo = cur.lo - delta, hi = cur.hi + delta;
  if (lo - lim.lo < delta) lo = lim.lo;
  if (lim.hi - hi < delta) hi = lim.hi;
  return {std::max(lo, lim.lo), std::min(hi, lim.hi)};
}

// partition_face (partition.hpp:156-212)
void band_face(const Face& face, const Net& main, Facing facing, const Params& p, std::vector<Panel>& out) {
  const Rect& r = face.r;
  int i0, i1;
  inplane(r.axis, i0, i1);
  const Box bb = bounding_box(main);
  const Span footA = clamp_to({bb.lo[i0], bb.hi[i0]}, r.a);
  const Span footB = clamp_to({bb.lo[i1], bb.hi[i1]}, r.b);
  const double step0 = std::max(p.p5, net_gap(r, main));
  std::vector<Rect> cells;
  auto emit = [&](Span sa, Span sb) {
    if (!(sa.len() > 0.0) || !(sb.len() > 0.0)) return;
    Rect strip = r;
    strip.a = sa;
    strip.b = sb;
    const double amax = area_bound(face.kind, facing, net_gap(strip, main), p);
    cells.clear();
    grid_strip(r, sa, sb, amax, p.aspect, cells);
    for (const Rect& c : cells) {
      Panel pn;
      pn.r = c;
      pn.kind = face.kind;
      pn.net = face.net;
      pn.regA = face.regA;
      pn.regB = face.regB;
      pn.area = c.area();
      pn.dist = net_gap(c, main);
      pn.facing = facing;
      out.push_back(pn);
    }
  };
  Span curA = grow_to(footA, r.a, step0), curB = grow_to(footB, r.b, step0);
  emit(curA, curB);
  double delta = step0;
  while (curA != r.a || curB != r.b) {
    delta *= 2.0;
    const Span nA = grow_to(curA, r.a, delta), nB = grow_to(curB, r.b, delta);
    emit(nA, Span{nB.lo, curB.lo});
    emit(nA, Span{curB.hi, nB.hi});
    emit(Span{nA.lo, curA.lo}, curB);
    emit(Span{curA.hi, nA.hi}, curB);
    curA = nA;
    curB = nB;
  }
}

PanelSet bucket_by_kind(std::vector<Panel>&& all, int main_net) {
  std::array<std::vector<Panel>, 4> by;
  for (Panel& pn : all) by[(int)pn.kind].push_back(pn);
  PanelSet ps;
  ps.main_net = main_net;
  ps.offset[0] = 0;
  for (int k = 0; k < 4; ++k) {
    ps.panels.insert(ps.panels.end(), by[k].begin(), by[k].end());
    ps.offset[k + 1] = ps.panels.size();
  }
  return ps;
}

}  // namespace

Facing face_facing(const Rect& r, const Net& main) {
  int i0, i1;
  inplane(r.axis, i0, i1);
  for (const Box& c : main.cells) {
    if (r.level != c.lo[r.axis] && r.level != c.hi[r.axis]) continue;
    if (r.a.lo >= c.lo[i0] && r.a.hi <= c.hi[i0] && r.b.lo >= c.lo[i1] && r.b.hi <= c.hi[i1]) return kOnMainNet;
  }
  const Box bb = bounding_box(main);
  const double centre = 0.5 * (bb.lo[r.axis] + bb.hi[r.axis]);
  return (centre - r.level) * r.nsign > 0 ? kFacing : kBack;
}

double area_bound(Kind k, Facing f, double d, const Params& p) {
  const double base = f == kBack ? p.p1 * p.p2 : p.p1;
  if (d <= p.p5) return base;
  const bool steep = k == kConductor || k == kDirichlet;
  return base * p.p3 * std::pow(d / p.p5, steep ? p.exp_dirichlet : p.exp_soft);
}

PanelSet partition_for_net(const Scene& s, int main_net, const Params& p) {
  p.check();
  const Net* main = s.net(main_net);
  if (!main) throw ValidationError("unknown main net id");
  std::vector<Panel> all;
  for (const Face& f : scene_faces(s)) band_face(f, *main, face_facing(f.r, *main), p, all);
  return bucket_by_kind(std::move(all), main_net);
}

std::vector<double> graded_edges(double lo, double hi, const GradedRule& g) {
  const double L = hi - lo;
  std::vector<double> side;
  double s = g.h0, used = 0.0;
  for (;;) {
    const double c = std::min(s, g.hmax);
    if (2.0 * (used + c) > L) break;
    side.push_back(c);
    used += c;
    s *= g.ratio;
  }
  std::vector<double> e{lo};
  double x = lo;
  for (double c : side) e.push_back(x += c);
  const double rem = L - 2.0 * used;
  if (rem > 1e-12 * L) {
    const double next = std::min(s, g.hmax);
    const int nmid = std::max(1, (int)std::ceil(rem / next - 1e-9));
    const double base = x;
    for (int k = 1; k < nmid; ++k) e.push_back(base + rem * k / nmid);
    x = base + rem;
    e.push_back(x);
  }
  for (size_t k = side.size(); k-- > 0;) e.push_back(x += side[k]);
  e.back() = hi;
  // drop zero-length cells produced by rounding at the join
  std::vector<double> out{e.front()};
  for (size_t k = 1; k < e.size(); ++k)
    if (e[k] > out.back()) out.push_back(e[k]);
  if (out.back() != hi) out.back() = hi;
  return out;
}

namespace {

PanelSet tensor_partition(const Scene& s, const std::function<std::vector<double>(double, double)>& edges) {
  std::vector<Panel> all;
  for (const Face& f : scene_faces(s)) {
    const std::vector<double> ea = edges(f.r.a.lo, f.r.a.hi), eb = edges(f.r.b.lo, f.r.b.hi);
    for (size_t ia = 0; ia + 1 < ea.size(); ++ia)
      for (size_t ib = 0; ib + 1 < eb.size(); ++ib) {
        Panel pn;
        pn.r = f.r;
        pn.r.a = Span{ea[ia], ea[ia + 1]};
        pn.r.b = Span{eb[ib], eb[ib + 1]};
        pn.kind = f.kind;
        pn.net = f.net;
        pn.regA = f.regA;
        pn.regB = f.regB;
        pn.area = pn.r.area();
        pn.dist = 0;
        pn.facing = kFacing;
        all.push_back(pn);
      }
  }
  return bucket_by_kind(std::move(all), -1);
}

}  // namespace

PanelSet partition_uniform(const Scene& s, double h) {
  if (!(h > 0)) throw ValidationError("uniform panel edge must be positive");
  return tensor_partition(s, [h](double lo, double hi) {
    const int n = std::max(1, (int)std::llround((hi - lo) / h));
    std::vector<double> e((size_t)n + 1);
    for (int k = 0; k <= n; ++k) e[(size_t)k] = k == n ? hi : lo + (hi - lo) * k / n;
    return e;
  });
}

PanelSet partition_graded(const Scene& s, const GradedRule& g) {
  if (!(g.h0 > 0) || !(g.ratio >= 1) || !(g.hmax >= g.h0)) throw ValidationError("bad graded rule");
  return tensor_partition(s, [&g](double lo, double hi) { return graded_edges(lo, hi, g); });
}

}  // namespace gbh

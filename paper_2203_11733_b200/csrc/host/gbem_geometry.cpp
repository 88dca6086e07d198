// gbem_geometry.cpp — scene validation and boundary-face extraction
// (semantics of proj/include/gbem/geometry.hpp:79-141, 226-324, 380-480).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>

#include "gbem_host.hpp"

namespace gbh {

double Rect::diameter() const { return std::hypot(a.len(), b.len()); }

const char* kind_name(Kind k) {
  static const char* names[4] = {"conductor", "dirichlet", "neumann", "interface"};
  return names[(int)k & 3];
}

namespace {

double sq_gap(double alo, double ahi, double blo, double bhi) {
  double g = std::max({blo - ahi, alo - bhi, 0.0});
  return g * g;
}

std::string num(double v) {
  char buf[32];
  std::snprintf(buf, sizeof buf, "%g", v);
  return buf;
}

std::string triple(const std::array<double, 3>& v) {
  return "(" + num(v[0]) + "," + num(v[1]) + "," + num(v[2]) + ")";
}

bool open_overlap(const Span& x, const Span& y) { return std::min(x.hi, y.hi) > std::max(x.lo, y.lo); }

Span meet(const Span& x, const Span& y) { return {std::max(x.lo, y.lo), std::min(x.hi, y.hi)}; }

bool interiors_meet(const Box& x, const Box& y) {
  for (int k = 0; k < 3; ++k)
    if (std::min(x.hi[k], y.hi[k]) <= std::max(x.lo[k], y.lo[k])) return false;
  return true;
}

// positiveAreaContact (geometry.hpp:112-125)
bool share_face_patch(const Box& x, const Box& y) {
  if (interiors_meet(x, y)) return false;
  for (int k = 0; k < 3; ++k) {
    if (x.hi[k] != y.lo[k] && y.hi[k] != x.lo[k]) continue;
    int i0, i1;
    inplane(k, i0, i1);
    if (open_overlap(x.extent(i0), y.extent(i0)) && open_overlap(x.extent(i1), y.extent(i1))) return true;
  }
  return false;
}

bool contains_closed(const Box& outer, const Box& c) {
  for (int k = 0; k < 3; ++k)
    if (c.lo[k] < outer.lo[k] || c.hi[k] > outer.hi[k]) return false;
  return true;
}

bool contains_strict(const Box& outer, const Box& c) {
  for (int k = 0; k < 3; ++k)
    if (c.lo[k] <= outer.lo[k] || c.hi[k] >= outer.hi[k]) return false;
  return true;
}

using Patch = std::array<Span, 2>;

// subtractCovers (geometry.hpp:380-401): left / right / bottom / top remainders.
std::vector<Patch> carve(const Patch& whole, const std::vector<Patch>& covers) {
  std::vector<Patch> cur{whole};
  for (const Patch& cv : covers) {
    std::vector<Patch> nxt;
    nxt.reserve(cur.size() + 3);
    for (const Patch& p : cur) {
      Span ia = meet(p[0], cv[0]), ib = meet(p[1], cv[1]);
      if (!ia.valid() || !ib.valid()) {
        nxt.push_back(p);
        continue;
      }
      if (p[0].lo < ia.lo) nxt.push_back({Span{p[0].lo, ia.lo}, p[1]});
      if (ia.hi < p[0].hi) nxt.push_back({Span{ia.hi, p[0].hi}, p[1]});
      if (p[1].lo < ib.lo) nxt.push_back({ia, Span{p[1].lo, ib.lo}});
      if (ib.hi < p[1].hi) nxt.push_back({ia, Span{ib.hi, p[1].hi}});
    }
    cur.swap(nxt);
  }
  return cur;
}

}  // namespace

double rect_gap(const Rect& x, const Rect& y) {
  double s = 0;
  for (int k = 0; k < 3; ++k) {
    Span ex = x.extent(k), ey = y.extent(k);
    s += sq_gap(ex.lo, ex.hi, ey.lo, ey.hi);
  }
  return std::sqrt(s);
}

double rect_box_gap(const Rect& r, const Box& c) {
  double s = 0;
  for (int k = 0; k < 3; ++k) {
    Span e = r.extent(k);
    double g = std::max({c.lo[k] - e.hi, e.lo - c.hi[k], 0.0});
    s += g * g;
  }
  return std::sqrt(s);
}

double net_gap(const Rect& r, const Net& n) {
  double d = std::numeric_limits<double>::infinity();
  for (const Box& c : n.cells) d = std::min(d, rect_box_gap(r, c));
  return d;
}

const Region* Scene::region(int id) const {
  for (const Region& r : regions)
    if (r.id == id) return &r;
  return nullptr;
}

const Net* Scene::net(int id) const {
  for (const Net& n : nets)
    if (n.id == id) return &n;
  return nullptr;
}

Scene make_scene(const Box& domain, std::vector<Region> regions, std::vector<Net> nets,
                 const std::array<int, 6>& bc, bool freespace) {
  Scene s;
  if (!domain.valid())
    throw ValidationError("domain box is degenerate: lo " + triple(domain.lo) + " hi " + triple(domain.hi));
  s.domain = domain;
  s.bc = bc;
  s.freespace = freespace;
  if (regions.empty()) throw ValidationError("scene has no dielectric regions");
  std::sort(regions.begin(), regions.end(), [](const Region& x, const Region& y) { return x.id < y.id; });
  double vol = 0;
  for (size_t i = 0; i < regions.size(); ++i) {
    const Region& r = regions[i];
    std::string tag = "region " + std::to_string(r.id);
    if (i && regions[i - 1].id == r.id) throw ValidationError("duplicate region id " + std::to_string(r.id));
    if (!r.box.valid()) throw ValidationError(tag + " box is degenerate");
    if (!(r.eps > 0)) throw ValidationError(tag + " relative permittivity must be positive");
    if (!contains_closed(domain, r.box)) throw ValidationError(tag + " extends outside the domain box");
    vol += r.box.volume();
  }
  for (size_t i = 0; i < regions.size(); ++i)
    for (size_t j = i + 1; j < regions.size(); ++j)
      if (interiors_meet(regions[i].box, regions[j].box))
        throw ValidationError("regions " + std::to_string(regions[i].id) + " and " +
                              std::to_string(regions[j].id) + " overlap");
  if (std::abs(vol - domain.volume()) > 1e-12 * domain.volume())
    throw ValidationError("regions do not tile the domain box (volume gap)");
  s.regions = std::move(regions);

  std::sort(nets.begin(), nets.end(), [](const Net& x, const Net& y) { return x.id < y.id; });
  for (size_t i = 0; i < nets.size(); ++i) {
    const Net& n = nets[i];
    std::string tag = "net " + std::to_string(n.id);
    if (i && nets[i - 1].id == n.id) throw ValidationError("duplicate net id " + std::to_string(n.id));
    if (n.cells.empty()) throw ValidationError(tag + " has no cuboids");
    for (const Box& c : n.cells)
      if (!c.valid()) throw ValidationError(tag + " has a degenerate cuboid");
    for (size_t a = 0; a < n.cells.size(); ++a)
      for (size_t b = a + 1; b < n.cells.size(); ++b)
        if (interiors_meet(n.cells[a], n.cells[b]))
          throw ValidationError(tag + " cuboids overlap (cells must be interior-disjoint)");
  }
  for (size_t i = 0; i < nets.size(); ++i)
    for (size_t j = i + 1; j < nets.size(); ++j)
      for (const Box& x : nets[i].cells)
        for (const Box& y : nets[j].cells) {
          std::string pair = "nets " + std::to_string(nets[i].id) + " and " + std::to_string(nets[j].id);
          if (interiors_meet(x, y)) throw ValidationError(pair + " overlap");
          if (share_face_patch(x, y))
            throw ValidationError(pair + " touch with positive contact area (shorted nets)");
        }
  for (const Net& n : nets) {
    int owner = -1;
    for (const Box& c : n.cells) {
      int hit = -1;
      for (const Region& r : s.regions)
        if (contains_strict(r.box, c)) hit = r.id;
      if (hit < 0)
        throw ValidationError("net " + std::to_string(n.id) +
                              " is not strictly interior to a single dielectric region");
      if (owner < 0) owner = hit;
      if (owner != hit)
        throw ValidationError("net " + std::to_string(n.id) + " straddles regions " + std::to_string(owner) +
                              " and " + std::to_string(hit));
    }
    s.region_of_net[n.id] = owner;
  }
  s.nets = std::move(nets);
  return s;
}

std::vector<Face> scene_faces(const Scene& s) {
  std::vector<Face> out;
  for (const Net& n : s.nets) {
    const int reg = s.region_of_net.at(n.id);
    for (size_t ci = 0; ci < n.cells.size(); ++ci) {
      const Box& cell = n.cells[ci];
      for (int axis = 0; axis < 3; ++axis) {
        int i0, i1;
        inplane(axis, i0, i1);
        for (int hi = 0; hi < 2; ++hi) {
          const double lvl = hi ? cell.hi[axis] : cell.lo[axis];
          Patch fp{cell.extent(i0), cell.extent(i1)};
          std::vector<Patch> covers;
          for (size_t oi = 0; oi < n.cells.size(); ++oi) {
            if (oi == ci) continue;
            const Box& o = n.cells[oi];
            if ((hi ? o.lo[axis] : o.hi[axis]) != lvl) continue;
            Patch op{o.extent(i0), o.extent(i1)};
            if (open_overlap(fp[0], op[0]) && open_overlap(fp[1], op[1])) covers.push_back(op);
          }
          for (const Patch& p : carve(fp, covers)) {
            Face f;
            f.r = Rect{axis, lvl, p[0], p[1], hi ? 1 : -1};
            f.kind = kConductor;
            f.net = n.id;
            f.regA = reg;
            out.push_back(f);
          }
        }
      }
    }
  }
  if (s.freespace) return out;
  for (const Region& reg : s.regions) {
    for (int axis = 0; axis < 3; ++axis) {
      int i0, i1;
      inplane(axis, i0, i1);
      for (int hi = 0; hi < 2; ++hi) {
        const double lvl = hi ? reg.box.hi[axis] : reg.box.lo[axis];
        const double dom = hi ? s.domain.hi[axis] : s.domain.lo[axis];
        Patch fp{reg.box.extent(i0), reg.box.extent(i1)};
        if (lvl == dom) {
          Face f;
          f.r = Rect{axis, lvl, fp[0], fp[1], hi ? -1 : 1};  // outer normals point into the domain
          f.kind = s.bc[2 * axis + hi] == 0 ? kDirichlet : kNeumann;
          f.regA = reg.id;
          out.push_back(f);
          continue;
        }
        for (const Region& nb : s.regions) {
          if (nb.id <= reg.id) continue;
          if ((hi ? nb.box.lo[axis] : nb.box.hi[axis]) != lvl) continue;
          Span ia = meet(fp[0], nb.box.extent(i0)), ib = meet(fp[1], nb.box.extent(i1));
          if (!ia.valid() || !ib.valid()) continue;
          Face f;
          f.r = Rect{axis, lvl, ia, ib, hi ? 1 : -1};
          f.kind = kInterface;
          f.regA = reg.id;
          f.regB = nb.id;
          out.push_back(f);
        }
      }
    }
  }
  return out;
}

}  // namespace gbh

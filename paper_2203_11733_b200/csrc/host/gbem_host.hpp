// gbem_host.hpp — C++ host side of the B200 GBEM extractor.
//
// Keeps the reference's scene-file input, panel-partition scheme and
// capacitance-matrix output (proj/include/gbem/{geometry,partition,model_io,
// extraction}.hpp) and drives the GPU through the C-ABI of include/gbem_gpu.h.
// Units: um.  Errors: ValidationError (exit 1) / NumericalError (exit 2), as
// proj/include/gbem/errors.hpp:10-20.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

struct gbem_ctx;

namespace gbh {

struct ValidationError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------- geometry
// Span / Rect / Cuboid semantics of geometry.hpp:21-130.
struct Span {
  double lo = 0, hi = 0;
  double len() const { return hi - lo; }
  double mid() const { return 0.5 * (lo + hi); }
  bool valid() const { return lo < hi; }
  bool operator==(const Span& o) const { return lo == o.lo && hi == o.hi; }
  bool operator!=(const Span& o) const { return !(*this == o); }
};

inline void inplane(int axis, int& i0, int& i1) {
  i0 = axis == 0 ? 1 : 0;
  i1 = axis == 2 ? 1 : 2;
}

struct Rect {
  int axis = 2;
  double level = 0;
  Span a, b;      // extents along the in-plane axes in axis-index order
  int nsign = 1;  // normal along +axis (+1) or -axis (-1)
  double area() const { return a.len() * b.len(); }
  Span extent(int k) const {
    if (k == axis) return {level, level};
    int i0, i1;
    inplane(axis, i0, i1);
    return k == i0 ? a : b;
  }
  double diameter() const;
  bool operator==(const Rect& o) const {
    return axis == o.axis && level == o.level && a == o.a && b == o.b && nsign == o.nsign;
  }
};

struct Box {
  std::array<double, 3> lo{0, 0, 0}, hi{0, 0, 0};
  bool valid() const { return lo[0] < hi[0] && lo[1] < hi[1] && lo[2] < hi[2]; }
  double volume() const { return (hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]); }
  Span extent(int k) const { return {lo[k], hi[k]}; }
  bool operator==(const Box& o) const { return lo == o.lo && hi == o.hi; }
};

double rect_gap(const Rect& x, const Rect& y);        // rectDistance (geometry.hpp:79-87)
double rect_box_gap(const Rect& r, const Box& c);     // rectCuboidDistance (geometry.hpp:133-141)

enum Kind : int { kConductor = 0, kDirichlet = 1, kNeumann = 2, kInterface = 3 };
const char* kind_name(Kind k);

struct Face {
  Rect r;
  Kind kind = kConductor;
  int net = -1, regA = -1, regB = -1;
};

struct Region {
  int id = -1;
  Box box;
  double eps = 1.0;
  bool operator==(const Region& o) const { return id == o.id && box == o.box && eps == o.eps; }
};

struct Net {
  int id = -1;
  std::vector<Box> cells;
  bool operator==(const Net& o) const { return id == o.id && cells == o.cells; }
};

// Outer face index 2*axis + hi, i.e. -x,+x,-y,+y,-z,+z; 0 dirichlet, 1 neumann.
struct Scene {
  Box domain;
  std::vector<Region> regions;  // ascending id
  std::vector<Net> nets;        // ascending id
  std::array<int, 6> bc{0, 0, 0, 0, 0, 0};
  std::map<int, int> region_of_net;
  bool freespace = false;  // extension: no outer boundary (conductors in free space)
  const Region* region(int id) const;
  const Net* net(int id) const;
  bool operator==(const Scene& o) const {
    return domain == o.domain && regions == o.regions && nets == o.nets && bc == o.bc &&
           region_of_net == o.region_of_net && freespace == o.freespace;
  }
};

double net_gap(const Rect& r, const Net& n);  // face_distance (geometry.hpp:226-230)

// build_scene (geometry.hpp:237-324): validates and sorts; throws ValidationError.
Scene make_scene(const Box& domain, std::vector<Region> regions, std::vector<Net> nets,
                 const std::array<int, 6>& bc, bool freespace = false);

// extract_faces (geometry.hpp:408-480): conductor faces (ascending net, axis,
// side) minus same-net covers, then outer and interface faces per region.
std::vector<Face> scene_faces(const Scene& s);

// ---------------------------------------------------------------- partition
// PartitionParams (partition.hpp:15-31).
struct Params {
  double p1 = 1.5, p2 = 4.0, p3 = 1.0, p5 = 1.0;
  double exp_dirichlet = 3.0, exp_soft = 2.0, aspect = 4.0;
  void check() const;
};

enum Facing : int { kOnMainNet = 0, kFacing = 1, kBack = 2 };

struct Panel {
  Rect r;
  Kind kind = kConductor;
  int net = -1, regA = -1, regB = -1;
  double area = 0, dist = 0;
  Facing facing = kFacing;
};

struct PanelSet {
  std::vector<Panel> panels;
  int main_net = -1;
  std::array<size_t, 5> offset{};  // class-contiguous [conductor, dirichlet, neumann, interface, end]
  size_t count(Kind k) const { return offset[(int)k + 1] - offset[(int)k]; }
};

Facing face_facing(const Rect& r, const Net& main);                   // classify_face (partition.hpp:60-76)
double area_bound(Kind k, Facing f, double d, const Params& p);       // max_area (partition.hpp:78-85)
// partition_scene (partition.hpp:214-245): graded banding toward the main net.
PanelSet partition_for_net(const Scene& s, int main_net, const Params& p);

// Net-independent partitions for the one-matrix / K-right-hand-side path
// ("net-independent mode").  Conductor faces only when the
// scene is free-space; outer faces get the same rule otherwise.
struct GradedRule {
  double h0 = 0.005;     // first cell at every face edge
  double ratio = 1.5;    // geometric growth toward the face interior
  double hmax = 0.05;    // cap
};
// 1-D graded cell edges on [lo, hi] (both ends start at h0).
std::vector<double> graded_edges(double lo, double hi, const GradedRule& g);
PanelSet partition_uniform(const Scene& s, double h);
PanelSet partition_graded(const Scene& s, const GradedRule& g);

// ---------------------------------------------------------------- model I/O
struct Model {
  Scene scene;
  Params params;
};
Model parse_model(const std::string& text);                          // model_io.hpp:127-204
std::string dump_model(const Scene& s, const Params& p);             // model_io.hpp:207-228
std::string read_file(const std::string& path);

// ---------------------------------------------------------------- extraction
constexpr double kEps0 = 8.854187817e-12;  // extraction.hpp:20
constexpr double kUnitScale = 1e-6;        // extraction.hpp:21

struct Options {
  int device = 0;
  std::string dump_matrix;  // matrix dump path (extraction.hpp:83-99 format)
  double rel_tol = 1e-8;
  int max_levels = 16;
  bool collocation = false;  // ExtractionOptions::baselineCollocation (extraction.hpp:110-114)
  int solver = 0;            // shared mode: 0 auto (PCG iff the context has several ranks), 1 direct, 2 PCG
  int jacobi_blocks = 1;     // PCG: Jacobi blocks per rank
  double pcg_tol = 1e-10;
};

struct RowDiag {
  size_t panels = 0;
  double seconds = 0, residual = 0, neutrality = -1;
  std::string method;
  bool converged = true;
};

struct Row {
  int main_net = -1;
  std::map<int, double> cap;
  double outer = 0;
  RowDiag diag;
};

struct CapMatrix {
  std::vector<int> ids;
  std::vector<Row> rows;
  double reciprocity = 0;
};

// capacitance_row / capacitance_matrix (extraction.hpp:106-184): per-main-net
// partition, GPU assembly + GPU Cholesky per row.
Row capacitance_row(gbem_ctx* ctx, const Scene& s, int main_net, const Params& p, const Options& o);
CapMatrix capacitance_matrix(gbem_ctx* ctx, const Scene& s, const Params& p, const Options& o);
// One panel set for all nets: one assembly, one factorisation, K right-hand sides.
CapMatrix capacitance_matrix_shared(gbem_ctx* ctx, const Scene& s, const PanelSet& ps, const Options& o);

struct Report {
  std::string version = "1.0.0";
  Params params;
  std::vector<int> ids;
  std::vector<Row> rows;
  double reciprocity = -1;
  std::string baseline;  // "" or "collocation" (model_io.hpp:236,274)
};
std::string to_csv(const Report& r);   // model_io.hpp:242-263
std::string to_json(const Report& r);  // model_io.hpp:266-299

void dump_matrix_file(const std::string& path, const std::vector<double>& A, size_t n);

// ---------------------------------------------------------------- BASELINE configs
// Seeded synthetic scenes of BASELINE.json configs 1-5 (DESIGN.md pins the
// unspecified geometry).  Panel lists are net-independent.
struct ConfigCase {
  std::string name;
  Scene scene;           // empty nets for config 5 (random panels)
  PanelSet panels;
  double eps = 3.9;
  int nets = 0;          // K
};
ConfigCase make_config(int id, uint64_t seed, double scale = 1.0);

}  // namespace gbh

// gbem_model_io.cpp — the reference's line-oriented scene format and reports
// (proj/include/gbem/model_io.hpp:28-299): same grammar, same error messages
// ("line N: ..."), canonical %.17g dump, CSV (%.9g, no timings, byte-stable)
// and JSON (diagnostics and wall times).  One extension statement:
// `freespace` drops the outer boundary (conductors in an unbounded medium),
// used by the net-independent BASELINE configs.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>

#include "gbem_host.hpp"

namespace gbh {

namespace {

std::vector<std::string> split_tokens(const std::string& line) {
  std::vector<std::string> t;
  std::string cur;
  for (char ch : line) {
    if (ch == '#') break;
    if (ch == ' ' || ch == '\t' || ch == '\r') {
      if (!cur.empty()) t.push_back(cur), cur.clear();
    } else {
      cur += ch;
    }
  }
  if (!cur.empty()) t.push_back(cur);
  return t;
}

struct LineError {
  int line;
  [[noreturn]] void operator()(const std::string& m) const {
    throw ValidationError("line " + std::to_string(line) + ": " + m);
  }
};

double to_number(const std::string& tok, const LineError& err, const char* what) {
  size_t used = 0;
  double v = 0;
  try {
    v = std::stod(tok, &used);
  } catch (...) {
    used = 0;
  }
  if (tok.empty() || used != tok.size()) err(std::string("expected ") + what + ", got '" + tok + "'");
  return v;
}

int to_id(const std::string& tok, const LineError& err, const char* what) {
  size_t used = 0;
  long v = 0;
  try {
    v = std::stol(tok, &used);
  } catch (...) {
    used = 0;
  }
  if (tok.empty() || used != tok.size()) err(std::string("expected ") + what + ", got '" + tok + "'");
  return (int)v;
}

std::array<double, 3> to_point(const std::string& tok, const char* key, const LineError& err) {
  const std::string head = std::string(key) + "(";
  auto bad = [&] { err("expected " + std::string(key) + "(x,y,z), got '" + tok + "'"); };
  if (tok.compare(0, head.size(), head) != 0 || tok.back() != ')') bad();
  const std::string body = tok.substr(head.size(), tok.size() - head.size() - 1);
  std::array<double, 3> v{};
  size_t at = 0;
  for (int i = 0; i < 3; ++i) {
    size_t comma = i < 2 ? body.find(',', at) : body.size();
    if (comma == std::string::npos) bad();
    v[(size_t)i] = to_number(body.substr(at, comma - at), err, "coordinate");
    at = comma + 1;
  }
  return v;
}

std::string fmt(const char* f, double v) {
  char buf[48];
  std::snprintf(buf, sizeof buf, f, v);
  return buf;
}
std::string g17(double v) { return fmt("%.17g", v); }
std::string g9(double v) { return fmt("%.9g", v); }

const char* kFaceNames[6] = {"-x", "+x", "-y", "+y", "-z", "+z"};

}  // namespace

Model parse_model(const std::string& text) {
  std::istringstream in(text);
  std::string line;
  int ln = 0;
  bool have_domain = false, freespace = false;
  Box domain;
  std::vector<Region> regions;
  std::vector<Net> nets;
  std::map<int, size_t> net_at;
  std::array<int, 6> bc{0, 0, 0, 0, 0, 0};
  Params pp;
  while (std::getline(in, line)) {
    ++ln;
    const LineError err{ln};
    const std::vector<std::string> t = split_tokens(line);
    if (t.empty()) continue;
    const std::string& key = t[0];
    if (key == "domain") {
      if (have_domain) err("duplicate domain");
      if (t.size() != 3) err("expected: domain lo(x,y,z) hi(x,y,z)");
      domain.lo = to_point(t[1], "lo", err);
      domain.hi = to_point(t[2], "hi", err);
      have_domain = true;
    } else if (key == "region") {
      if (t.size() == 4 && t[2].rfind("lo(", 0) == 0) err("region " + t[1] + ": missing permittivity");
      if (t.size() != 5) err("expected: region <id> <eps> lo(x,y,z) hi(x,y,z)");
      Region r;
      r.id = to_id(t[1], err, "region id");
      if (t[2].rfind("lo(", 0) == 0) err("region " + t[1] + ": missing permittivity");
      r.eps = to_number(t[2], err, "permittivity");
      r.box.lo = to_point(t[3], "lo", err);
      r.box.hi = to_point(t[4], "hi", err);
      regions.push_back(r);
    } else if (key == "net") {
      if (t.size() != 5 || t[2] != "cuboid") err("expected: net <id> cuboid lo(x,y,z) hi(x,y,z)");
      const int id = to_id(t[1], err, "net id");
      Box c;
      c.lo = to_point(t[3], "lo", err);
      c.hi = to_point(t[4], "hi", err);
      auto it = net_at.find(id);
      if (it == net_at.end()) {
        net_at[id] = nets.size();
        nets.push_back(Net{id, {c}});
      } else {
        nets[it->second].cells.push_back(c);
      }
    } else if (key == "bc") {
      if (t.size() != 3) err("expected: bc <face> <dirichlet|neumann>");
      int idx = -1;
      for (int k = 0; k < 6; ++k)
        if (t[1] == kFaceNames[k]) idx = k;
      if (idx < 0) err("expected face in {+x,-x,+y,-y,+z,-z}, got '" + t[1] + "'");
      if (t[2] == "dirichlet")
        bc[(size_t)idx] = 0;
      else if (t[2] == "neumann")
        bc[(size_t)idx] = 1;
      else
        err("expected boundary type dirichlet or neumann, got '" + t[2] + "'");
    } else if (key == "params") {
      if (t.size() != 5) err("expected: params <p1> <p2> <p3> <p5>");
      pp.p1 = to_number(t[1], err, "p1");
      pp.p2 = to_number(t[2], err, "p2");
      pp.p3 = to_number(t[3], err, "p3");
      pp.p5 = to_number(t[4], err, "p5");
    } else if (key == "freespace") {
      if (t.size() != 1) err("expected: freespace");
      freespace = true;
    } else {
      err("unknown key '" + key + "'");
    }
  }
  if (!have_domain) throw ValidationError("scene file has no domain line");
  pp.check();
  Model m;
  m.scene = make_scene(domain, regions, nets, bc, freespace);
  m.params = pp;
  return m;
}

std::string dump_model(const Scene& s, const Params& p) {
  auto pt = [](const char* key, const std::array<double, 3>& v) {
    return std::string(key) + "(" + g17(v[0]) + "," + g17(v[1]) + "," + g17(v[2]) + ")";
  };
  std::ostringstream o;
  o << "domain " << pt("lo", s.domain.lo) << " " << pt("hi", s.domain.hi) << "\n";
  for (const Region& r : s.regions)
    o << "region " << r.id << " " << g17(r.eps) << " " << pt("lo", r.box.lo) << " " << pt("hi", r.box.hi) << "\n";
  for (const Net& n : s.nets)
    for (const Box& c : n.cells) o << "net " << n.id << " cuboid " << pt("lo", c.lo) << " " << pt("hi", c.hi) << "\n";
  for (int k = 0; k < 6; ++k) o << "bc " << kFaceNames[k] << " " << (s.bc[(size_t)k] ? "neumann" : "dirichlet") << "\n";
  o << "params " << g17(p.p1) << " " << g17(p.p2) << " " << g17(p.p3) << " " << g17(p.p5) << "\n";
  if (s.freespace) o << "freespace\n";
  return o.str();
}

std::string read_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw ValidationError("cannot open input file: " + path);
  std::ostringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

std::string to_csv(const Report& r) {
  std::ostringstream o;
  o << "# gbem " << r.version << "\n";
  o << "# params p1=" << g9(r.params.p1) << " p2=" << g9(r.params.p2) << " p3=" << g9(r.params.p3)
    << " p5=" << g9(r.params.p5) << "\n";
  o << "# panels";
  for (const Row& row : r.rows) o << " net" << row.main_net << "=" << row.diag.panels;
  o << "\n# method";
  for (const Row& row : r.rows) o << " net" << row.main_net << "=" << row.diag.method;
  o << "\nnet";
  for (int id : r.ids) o << "," << id;
  o << "\n";
  for (const Row& row : r.rows) {
    o << row.main_net;
    for (int id : r.ids) o << "," << g9(row.cap.at(id));
    o << "\n";
  }
  return o.str();
}

std::string to_json(const Report& r) {
  std::ostringstream o;
  o << "{\n  \"tool\": \"gbem\",\n  \"version\": \"" << r.version << "\",\n";
  o << "  \"params\": {\"p1\": " << g9(r.params.p1) << ", \"p2\": " << g9(r.params.p2) << ", \"p3\": "
    << g9(r.params.p3) << ", \"p5\": " << g9(r.params.p5) << "},\n";
  if (!r.baseline.empty()) o << "  \"baseline\": \"" << r.baseline << "\",\n";
  o << "  \"netIds\": [";
  for (size_t i = 0; i < r.ids.size(); ++i) o << (i ? ", " : "") << r.ids[i];
  o << "],\n  \"rows\": [\n";
  for (size_t i = 0; i < r.rows.size(); ++i) {
    const Row& row = r.rows[i];
    o << "    {\"net\": " << row.main_net << ", \"panels\": " << row.diag.panels << ", \"method\": \""
      << row.diag.method << "\", \"residual\": " << g9(row.diag.residual) << ", \"neutrality\": "
      << g9(row.diag.neutrality) << ", \"outerCharge\": " << g9(row.outer) << ", \"seconds\": "
      << g9(row.diag.seconds) << ", \"capacitance\": {";
    bool first = true;
    for (const auto& kv : row.cap) {
      o << (first ? "" : ", ") << "\"" << kv.first << "\": " << g9(kv.second);
      first = false;
    }
    o << "}}" << (i + 1 < r.rows.size() ? "," : "") << "\n";
  }
  o << "  ],\n  \"reciprocityDefect\": " << g9(r.reciprocity) << "\n}\n";
  return o.str();
}

void dump_matrix_file(const std::string& path, const std::vector<double>& A, size_t n) {
  // extraction.hpp:83-99: u64 LE n, then n^2 f64 LE row-major
  std::ofstream f(path, std::ios::binary);
  if (!f) throw ValidationError("cannot open matrix dump path: " + path);
  auto le = [&f](uint64_t v) {
    unsigned char b[8];
    for (int i = 0; i < 8; ++i) b[i] = (unsigned char)(v >> (8 * i));
    f.write(reinterpret_cast<const char*>(b), 8);
  };
  le((uint64_t)n);
  for (size_t k = 0; k < n * n; ++k) {
    uint64_t bits;
    std::memcpy(&bits, &A[k], 8);
    le(bits);
  }
}

}  // namespace gbh

// gbem_host_capi.cpp — extern "C" surface of the C++ host (include/gbem_host.h).
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <thread>

#include "../../../include/gbem_gpu.h"
#include "../../../include/gbem_host.h"
#include "gbem_host.hpp"

struct gbem_model {
  gbh::Scene scene;
  gbh::Params params;
  gbh::PanelSet panels;
  bool has_config = false;
  gbh::PanelSet config_panels;
};

namespace {

void put_err(char* err, int len, const std::string& m) {
  if (err && len > 0) {
    std::strncpy(err, m.c_str(), (size_t)len - 1);
    err[len - 1] = 0;
  }
}

template <class F>
int guarded(char* err, int len, F&& f) {
  try {
    f();
    return 0;
  } catch (const gbh::ValidationError& e) {
    put_err(err, len, e.what());
    return 1;
  } catch (const gbh::NumericalError& e) {
    put_err(err, len, e.what());
    return 2;
  } catch (const std::exception& e) {
    put_err(err, len, e.what());
    return 3;
  }
}

void copy_out(const std::string& s, char* buf, int64_t cap, int64_t* len) {
  if (len) *len = (int64_t)s.size();
  if (buf && cap > (int64_t)s.size()) std::memcpy(buf, s.c_str(), s.size() + 1);
}

}  // namespace

extern "C" {

int gbem_model_parse(const char* text, gbem_model** out, char* err, int errlen) {
  if (!out || !text) return 1;
  *out = nullptr;
  return guarded(err, errlen, [&] {
    auto m = std::make_unique<gbem_model>();
    gbh::Model pm = gbh::parse_model(text);
    m->scene = pm.scene;
    m->params = pm.params;
    *out = m.release();
  });
}

int gbem_model_config(int config, uint64_t seed, double scale, gbem_model** out, char* err, int errlen) {
  if (!out) return 1;
  *out = nullptr;
  return guarded(err, errlen, [&] {
    if (!(scale > 0)) throw gbh::ValidationError("scale must be positive");
    gbh::ConfigCase cc = gbh::make_config(config, seed, scale);
    auto m = std::make_unique<gbem_model>();
    m->scene = cc.scene;
    m->config_panels = cc.panels;
    m->panels = cc.panels;
    m->has_config = true;
    *out = m.release();
  });
}

void gbem_model_free(gbem_model* m) { delete m; }

int64_t gbem_model_dump(const gbem_model* m, char* buf, int64_t cap) {
  if (!m) return -1;
  if (m->scene.regions.empty()) return 0;
  std::string s = gbh::dump_model(m->scene, m->params);
  int64_t len = 0;
  copy_out(s, buf, cap, &len);
  return len;
}

int gbem_model_nets(const gbem_model* m, int32_t* ids, int cap) {
  if (!m) return -1;
  int k = 0;
  for (const gbh::Net& n : m->scene.nets) {
    if (ids && k < cap) ids[k] = n.id;
    ++k;
  }
  return k;
}

int gbem_model_info(const gbem_model* m, int32_t* nregions, int32_t* nfaces, double* eps_r, int32_t* freespace) {
  if (!m) return 1;
  if (nregions) *nregions = (int32_t)m->scene.regions.size();
  if (nfaces) *nfaces = m->scene.regions.empty() ? 0 : (int32_t)gbh::scene_faces(m->scene).size();
  if (eps_r) *eps_r = m->scene.regions.empty() ? 1.0 : m->scene.regions.front().eps;
  if (freespace) *freespace = m->scene.freespace ? 1 : 0;
  return 0;
}

int gbem_model_regions(const gbem_model* m, int32_t* ids, double* eps, int cap) {
  if (!m) return -1;
  const int k = (int)m->scene.regions.size();
  for (int i = 0; i < k && i < cap; ++i) {
    if (ids) ids[i] = m->scene.regions[(size_t)i].id;
    if (eps) eps[i] = m->scene.regions[(size_t)i].eps;
  }
  return k;
}

int gbem_model_params(const gbem_model* m, double p[4]) {
  if (!m || !p) return 1;
  p[0] = m->params.p1;
  p[1] = m->params.p2;
  p[2] = m->params.p3;
  p[3] = m->params.p5;
  return 0;
}

int gbem_model_set_params(gbem_model* m, const double p[4], char* err, int errlen) {
  if (!m || !p) return 1;
  return guarded(err, errlen, [&] {
    gbh::Params q = m->params;
    q.p1 = p[0];
    q.p2 = p[1];
    q.p3 = p[2];
    q.p5 = p[3];
    q.check();
    m->params = q;
  });
}

int64_t gbem_model_partition(gbem_model* m, int mode, int32_t main_net, const double* args, char* err,
                             int errlen) {
  if (!m) return -1;
  int rc = guarded(err, errlen, [&] {
    switch (mode) {
      case 0:
        m->panels = gbh::partition_for_net(m->scene, main_net, m->params);
        break;
      case 1:
        if (!m->has_config) throw gbh::ValidationError("model has no config panel set");
        m->panels = m->config_panels;
        break;
      case 2:
        if (!args) throw gbh::ValidationError("uniform partition needs the panel edge");
        m->panels = gbh::partition_uniform(m->scene, args[0]);
        break;
      case 3: {
        if (!args) throw gbh::ValidationError("graded partition needs h0, ratio, hmax");
        gbh::GradedRule g{args[0], args[1], args[2]};
        m->panels = gbh::partition_graded(m->scene, g);
        break;
      }
      default:
        throw gbh::ValidationError("unknown partition mode");
    }
  });
  return rc ? -1 : (int64_t)m->panels.panels.size();
}

int gbem_model_panels(const gbem_model* m, uint8_t* axis, double* level, double* a0, double* a1, double* b0,
                      double* b1, int32_t* nsign, int32_t* kind, int32_t* net, int32_t* region_a,
                      int32_t* region_b, double* area, double* dist, int32_t* facing) {
  if (!m) return 1;
  size_t k = 0;
  for (const gbh::Panel& p : m->panels.panels) {
    if (axis) axis[k] = (uint8_t)p.r.axis;
    if (level) level[k] = p.r.level;
    if (a0) a0[k] = p.r.a.lo;
    if (a1) a1[k] = p.r.a.hi;
    if (b0) b0[k] = p.r.b.lo;
    if (b1) b1[k] = p.r.b.hi;
    if (nsign) nsign[k] = p.r.nsign;
    if (kind) kind[k] = (int32_t)p.kind;
    if (net) net[k] = p.net;
    if (region_a) region_a[k] = p.regA;
    if (region_b) region_b[k] = p.regB;
    if (area) area[k] = p.area;
    if (dist) dist[k] = p.dist;
    if (facing) facing[k] = (int32_t)p.facing;
    ++k;
  }
  return 0;
}

namespace {

// NCCL ranks for the sharded shared-mode solve: rank 0 writes the unique id to
// `path` (atomically, through a rename), the other ranks poll for it.
void attach_ranks(gbem_ctx* ctx, int nranks, int rank, const char* path) {
  if (!path || !*path) throw gbh::ValidationError("several ranks need an NCCL id file");
  if (rank < 0 || rank >= nranks) throw gbh::ValidationError("rank out of range");
  std::vector<char> id(GBEM_NCCL_UNIQUE_ID_BYTES);
  if (rank == 0) {
    if (gbem_nccl_unique_id(id.data()) != GBEM_OK) throw std::runtime_error("ncclGetUniqueId failed");
    const std::string tmp = std::string(path) + ".tmp";
    {
      std::ofstream f(tmp, std::ios::binary);
      f.write(id.data(), (std::streamsize)id.size());
      if (!f) throw std::runtime_error("cannot write " + tmp);
    }
    if (std::rename(tmp.c_str(), path) != 0) throw std::runtime_error(std::string("cannot rename to ") + path);
  } else {
    for (int t = 0;; ++t) {
      std::ifstream f(path, std::ios::binary);
      if (f && f.read(id.data(), (std::streamsize)id.size()) && f.gcount() == (std::streamsize)id.size()) break;
      if (t > 12000) throw std::runtime_error(std::string("timed out waiting for ") + path);
      std::this_thread::sleep_for(std::chrono::milliseconds(10));
    }
  }
  if (gbem_ctx_init_nccl(ctx, nranks, rank, id.data()) != GBEM_OK)
    throw std::runtime_error(std::string("NCCL: ") + gbem_last_error(ctx));
}

}  // namespace

int gbem_model_extract(const gbem_model* m, const gbem_extract_opts* o, char* csv, int64_t csv_cap,
                       int64_t* csv_len, char* json, int64_t json_cap, int64_t* json_len, char* err,
                       int errlen) {
  if (!m || !o) return 1;
  gbem_ctx* ctx = nullptr;
  int crc = gbem_ctx_create(o->device, &ctx);
  if (crc != GBEM_OK) {
    put_err(err, errlen, ctx ? gbem_last_error(ctx) : "context creation failed");
    gbem_ctx_destroy(ctx);
    return 3;
  }
  int rc = guarded(err, errlen, [&] {
    if (o->nranks > 1) attach_ranks(ctx, o->nranks, o->rank, o->nccl_id_file);
    gbh::Options opt;
    opt.device = o->device;
    opt.solver = o->solver;
    opt.jacobi_blocks = o->jacobi_blocks > 0 ? o->jacobi_blocks : 1;
    if (o->pcg_tol > 0) opt.pcg_tol = o->pcg_tol;
    if (o->rel_tol > 0) opt.rel_tol = o->rel_tol;
    if (o->max_levels > 0) opt.max_levels = o->max_levels;
    if (o->dump_matrix) opt.dump_matrix = o->dump_matrix;
    opt.collocation = o->collocation != 0;
    gbh::Report rep;
    if (opt.collocation) rep.baseline = "collocation";
    rep.params = m->params;
    for (const gbh::Net& n : m->scene.nets) rep.ids.push_back(n.id);
    if (o->mode == 1) {
      gbh::CapMatrix cm = gbh::capacitance_matrix_shared(ctx, m->scene, m->panels, opt);
      if (o->net >= 0) {
        for (const gbh::Row& r : cm.rows)
          if (r.main_net == o->net) rep.rows.push_back(r);
        if (rep.rows.empty()) throw gbh::ValidationError("unknown main net id");
      } else {
        rep.rows = cm.rows;
        rep.reciprocity = cm.reciprocity;
      }
    } else if (o->net >= 0) {
      rep.rows.push_back(gbh::capacitance_row(ctx, m->scene, o->net, m->params, opt));
    } else {
      gbh::CapMatrix cm = gbh::capacitance_matrix(ctx, m->scene, m->params, opt);
      rep.rows = cm.rows;
      rep.reciprocity = cm.reciprocity;
    }
    for (size_t r = 0; r < rep.rows.size(); ++r) {
      if (o->cap_out)
        for (size_t k = 0; k < rep.ids.size(); ++k) o->cap_out[r * rep.ids.size() + k] = rep.rows[r].cap.at(rep.ids[k]);
      if (o->outer_out) o->outer_out[r] = rep.rows[r].outer;
    }
    copy_out(gbh::to_csv(rep), csv, csv_cap, csv_len);
    copy_out(gbh::to_json(rep), json, json_cap, json_len);
  });
  gbem_ctx_destroy(ctx);
  return rc;
}

}  // extern "C"

// gbem_cli.cpp — command-line driver (the reference's `gbem extract|validate`,
// proj/include/gbem/cli.hpp:18-128) on the B200 path.  Exit codes: 0 success,
// 1 input/validation error, 2 numerical failure, 3 CUDA/runtime failure.
//
//   gbem extract --input F [--net N | --all] [--p1 X] [--p2 X] [--p3 X] [--p5 X]
//                [--format csv|json] [--output P] [--dump-matrix P]
//                [--mode per-net|shared] [--uniform H | --graded H0,R,HMAX] [--device D]
//                [--baseline collocation]
//                [--solver auto|direct|pcg] [--jacobi-blocks B] [--pcg-tol X]
//                [--ranks N --rank R --nccl-id FILE]   (shared mode on row-block shards, one process per GPU)
//   gbem validate --input F
//   gbem kernels selftest [--pairs N] [--seed S] [--device D]   (cli.hpp:48-75, on the GPU)
//   gbem config --id N [--seed S] [--scale X]      (prints the config scene + panel count)
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "../../../include/gbem_gpu.h"
#include "../../../include/gbem_host.h"
#include "gbem_host.hpp"

namespace {

int usage(const char* msg) {
  std::cerr << "input error: " << msg << "\n"
            << "usage: gbem extract --input F [--net N|--all] [--format csv|json] [--output P]\n"
            << "       gbem validate --input F\n"
            << "       gbem kernels selftest [--pairs N] [--seed S] [--device D]\n"
            << "       gbem config --id N [--seed S] [--scale X]\n";
  return 1;
}

bool num(const std::string& s, double& v) {
  try {
    size_t k = 0;
    v = std::stod(s, &k);
    return k == s.size();
  } catch (...) {
    return false;
  }
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage("missing subcommand");
  std::string cmd = argv[1];
  std::vector<std::string> a(argv + 2, argv + argc);
  auto value = [&](size_t& i, std::string& out) {
    if (i + 1 >= a.size()) return false;
    out = a[++i];
    return true;
  };
  char err[1024] = {0};
  if (cmd == "validate") {
    std::string in;
    for (size_t i = 0; i < a.size(); ++i) {
      if (a[i] == "--input" && value(i, in)) continue;
      return usage(("unknown option " + a[i]).c_str());
    }
    if (in.empty()) return usage("--input is required");
    try {
      gbh::Model m = gbh::parse_model(gbh::read_file(in));
      std::cout << "ok: " << m.scene.nets.size() << " nets, " << m.scene.regions.size() << " regions, "
                << gbh::scene_faces(m.scene).size() << " boundary faces\n";
      return 0;
    } catch (const gbh::ValidationError& e) {
      std::cerr << "input error: " << e.what() << "\n";
      return 1;
    }
  }
  if (cmd == "kernels") {
    // run_selftest (selftest.hpp:184-245) on the GPU; exit 2 when a class fails (cli.hpp:70-75)
    if (a.empty() || a[0] != "selftest") return usage("expected: kernels selftest");
    double pairs = 500, seed = 20260817, dev = 0;
    std::string v;
    for (size_t i = 1; i < a.size(); ++i) {
      if (a[i] == "--pairs" && value(i, v) && num(v, pairs) && pairs >= 1) continue;
      if (a[i] == "--seed" && value(i, v) && num(v, seed)) continue;
      if (a[i] == "--device" && value(i, v) && num(v, dev)) continue;
      return usage(("bad option " + a[i]).c_str());
    }
    gbem_ctx* ctx = nullptr;
    if (gbem_ctx_create((int)dev, &ctx) != GBEM_OK) {
      std::cerr << "runtime error: " << gbem_last_error(ctx) << "\n";
      gbem_ctx_destroy(ctx);
      return 3;
    }
    gbem_selftest_case cases[10];
    int32_t nc = 0;
    int rc = gbem_selftest(ctx, (int32_t)pairs, (uint64_t)seed, nullptr, cases, &nc);
    if (rc) {
      std::cerr << (rc == GBEM_EINVAL ? "input error: " : "runtime error: ") << gbem_last_error(ctx) << "\n";
      gbem_ctx_destroy(ctx);
      return rc;
    }
    gbem_ctx_destroy(ctx);
    bool pass = true;
    for (int c = 0; c < nc; ++c) {
      char buf[160];
      std::snprintf(buf, sizeof(buf), "%-24s pairs=%-5d worst_rel=%.3e tol=%.0e  %s", cases[c].name, cases[c].pairs,
                    cases[c].worst_rel, cases[c].tol, cases[c].pass ? "PASS" : "FAIL");
      std::cout << buf << "\n";
      pass = pass && cases[c].pass;
    }
    if (!pass) {
      std::cerr << "selftest failed: kernel/oracle disagreement above threshold\n";
      return 2;
    }
    return 0;
  }
  if (cmd == "config") {
    double id = 2, seed = 1, scale = 1;
    std::string v;
    for (size_t i = 0; i < a.size(); ++i) {
      if (a[i] == "--id" && value(i, v) && num(v, id)) continue;
      if (a[i] == "--seed" && value(i, v) && num(v, seed)) continue;
      if (a[i] == "--scale" && value(i, v) && num(v, scale)) continue;
      return usage(("bad option " + a[i]).c_str());
    }
    gbem_model* m = nullptr;
    int rc = gbem_model_config((int)id, (uint64_t)seed, scale, &m, err, sizeof err);
    if (rc) {
      std::cerr << "input error: " << err << "\n";
      return rc;
    }
    int64_t len = gbem_model_dump(m, nullptr, 0);
    std::string text((size_t)len + 1, '\0');
    gbem_model_dump(m, &text[0], len + 1);
    text.resize((size_t)len);
    std::cout << text << "# panels " << gbem_model_partition(m, 1, -1, nullptr, err, sizeof err) << "\n";
    gbem_model_free(m);
    return 0;
  }
  if (cmd != "extract") return usage(("unknown subcommand " + cmd).c_str());
  std::string in, out, format = "csv", dump, mode = "per-net", v, baseline, solver = "auto", ncclid;
  double p[4] = {-1, -1, -1, -1}, netd = -1, dev = 0, uni = -1, ranks = 1, rank = 0, jblocks = 1, ptol = 0;
  double graded[3] = {-1, -1, -1};
  bool all = false, have_net = false;
  for (size_t i = 0; i < a.size(); ++i) {
    const std::string& k = a[i];
    if (k == "--input" && value(i, in)) continue;
    if (k == "--output" && value(i, out)) continue;
    if (k == "--format" && value(i, format) && (format == "csv" || format == "json")) continue;
    if (k == "--dump-matrix" && value(i, dump)) continue;
    if (k == "--mode" && value(i, mode) && (mode == "per-net" || mode == "shared")) continue;
    if (k == "--baseline" && value(i, baseline) && baseline == "collocation") continue;  // cli.hpp:37-38
    if (k == "--solver" && value(i, solver) && (solver == "auto" || solver == "direct" || solver == "pcg")) continue;
    if (k == "--jacobi-blocks" && value(i, v) && num(v, jblocks) && jblocks >= 1) continue;
    if (k == "--pcg-tol" && value(i, v) && num(v, ptol) && ptol > 0) continue;
    if (k == "--ranks" && value(i, v) && num(v, ranks) && ranks >= 1) continue;
    if (k == "--rank" && value(i, v) && num(v, rank) && rank >= 0) continue;
    if (k == "--nccl-id" && value(i, ncclid)) continue;
    if (k == "--all") {
      all = true;
      continue;
    }
    if (k == "--net" && value(i, v) && num(v, netd)) {
      have_net = true;
      continue;
    }
    if (k == "--device" && value(i, v) && num(v, dev)) continue;
    if (k == "--uniform" && value(i, v) && num(v, uni)) continue;
    if (k == "--graded" && value(i, v) &&
        std::sscanf(v.c_str(), "%lf,%lf,%lf", &graded[0], &graded[1], &graded[2]) == 3)
      continue;
    bool matched = false;
    for (int q = 0; q < 4; ++q) {
      static const char* names[4] = {"--p1", "--p2", "--p3", "--p5"};
      if (k == names[q] && value(i, v) && num(v, p[q])) matched = true;
    }
    if (matched) continue;
    return usage(("bad option " + k).c_str());
  }
  if (in.empty()) return usage("--input is required");
  if (all && have_net) {
    std::cerr << "input error: --net and --all are mutually exclusive\n";
    return 1;
  }
  std::string text;
  try {
    text = gbh::read_file(in);
  } catch (const gbh::ValidationError& e) {
    std::cerr << "input error: " << e.what() << "\n";
    return 1;
  }
  gbem_model* m = nullptr;
  int rc = gbem_model_parse(text.c_str(), &m, err, sizeof err);
  if (rc) {
    std::cerr << "input error: " << err << "\n";
    return rc;
  }
  double cur[4];
  gbem_model_params(m, cur);
  for (int q = 0; q < 4; ++q)
    if (p[q] > 0) cur[q] = p[q];
  if ((rc = gbem_model_set_params(m, cur, err, sizeof err))) {
    std::cerr << "input error: " << err << "\n";
    gbem_model_free(m);
    return rc;
  }
  gbem_extract_opts o{};
  o.device = (int32_t)dev;
  o.mode = mode == "shared" ? 1 : 0;
  o.net = have_net ? (int32_t)netd : -1;
  o.dump_matrix = dump.empty() ? nullptr : dump.c_str();
  o.collocation = baseline == "collocation" ? 1 : 0;
  o.solver = solver == "direct" ? 1 : (solver == "pcg" ? 2 : 0);
  o.jacobi_blocks = (int32_t)jblocks;
  o.pcg_tol = ptol;
  o.nranks = (int32_t)ranks;
  o.rank = (int32_t)rank;
  o.nccl_id_file = ncclid.empty() ? nullptr : ncclid.c_str();
  if (o.nranks > 1 && o.mode != 1) {
    std::cerr << "input error: --ranks needs --mode shared\n";
    gbem_model_free(m);
    return 1;
  }
  if (o.collocation && o.mode == 1) {
    std::cerr << "input error: --baseline collocation runs per net (--mode per-net)\n";
    gbem_model_free(m);
    return 1;
  }
  if (o.mode == 1) {
    int64_t n = -1;
    if (uni > 0)
      n = gbem_model_partition(m, 2, -1, &uni, err, sizeof err);
    else if (graded[0] > 0)
      n = gbem_model_partition(m, 3, -1, graded, err, sizeof err);
    else
      n = -2;
    if (n == -2) {
      std::cerr << "input error: --mode shared needs --uniform H or --graded H0,R,HMAX\n";
      gbem_model_free(m);
      return 1;
    }
    if (n < 0) {
      std::cerr << "input error: " << err << "\n";
      gbem_model_free(m);
      return 1;
    }
  }
  int64_t csv_len = 0, json_len = 0;
  std::string csv(1 << 20, '\0'), json(1 << 20, '\0');
  rc = gbem_model_extract(m, &o, &csv[0], (int64_t)csv.size(), &csv_len, &json[0], (int64_t)json.size(), &json_len,
                          err, sizeof err);
  if (rc == 0 && (csv_len >= (int64_t)csv.size() || json_len >= (int64_t)json.size())) {
    csv.assign((size_t)csv_len + 1, '\0');
    json.assign((size_t)json_len + 1, '\0');
    rc = gbem_model_extract(m, &o, &csv[0], csv_len + 1, &csv_len, &json[0], json_len + 1, &json_len, err,
                            sizeof err);
  }
  if (rc == 0) {
    csv.resize((size_t)csv_len);
    json.resize((size_t)json_len);
  }
  gbem_model_free(m);
  if (rc == 1) {
    std::cerr << "input error: " << err << "\n";
    return 1;
  }
  if (rc == 2) {
    std::cerr << "numerical error: " << err << "\n";
    return 2;
  }
  if (rc) {
    std::cerr << "error: " << err << "\n";
    return 3;
  }
  if (o.nranks > 1 && o.rank != 0) return 0;  // every rank holds the same matrix; rank 0 reports
  const std::string& report = format == "json" ? json : csv;
  if (out.empty()) {
    std::cout << report;
  } else {
    std::ofstream f(out, std::ios::binary);
    if (!f) {
      std::cerr << "input error: cannot open output file: " << out << "\n";
      return 1;
    }
    f << report;
  }
  return 0;
}

// tests/cpp/compat_test.cpp -- TEST INFRASTRUCTURE: the heplan-side binding
// (paper_2604_03425_b200/csrc/heplan_compat.hpp) compiled against the
// UNMODIFIED reference headers (/root/reference/proj/include) and libaegis.
//
//   compat_test plan <dir>   no device: the reference lowers config 1 (FFN,
//                            N=2^16, T=128) and a block (N=2^11, T=32);
//                            heplan_compat ingests each in-memory HeOpGraph
//                            (aegis_graph_from_ops) and dumps it; libaegis'
//                            own lowering is dumped beside it.  Exit 0 iff
//                            every pair is identical.
//   compat_test run          device 0: Executor::exec_sequential on the
//                            reference-lowered FFN at N=2^10, T=8; prints one
//                            bundle hash per line (the pytest compares them
//                            with the CPU oracle on the same graph).
//
// he_ir.hpp holds `const CtBundle&` across make_bundle(); as in
// oracle/ref_shim.cpp the lowering's vectors are reserved before run() so the
// emitted graph is the reference's, without editing the header.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>

#define private public
#include "heplan/ckks.hpp"
#include "heplan/graph.hpp"
#include "heplan/he_ir.hpp"
#undef private

#include "paper_2604_03425_b200/csrc/heplan_compat.hpp"

using namespace heplan;

namespace {

struct Lowered {
  CkksProfile prof;
  PackingLayout lay;
  TransformerConfig cfg;
  HeOpGraph he;
};

Lowered lower(uint32_t n, uint64_t tokens, int kind) {
  Lowered r;
  r.prof = CkksProfile{n, n / 2, 35, 4, 8, 14};
  r.prof.validate();
  r.lay = PackingLayout{64, 768, 64};
  r.lay.validate(r.prof);
  r.cfg.layer_count = 1;
  AppGraph app;
  if (kind == 0) {
    app = build_transformer_graph(r.cfg, r.prof, tokens);
  } else {  // ffn1 -> gelu -> ffn2 at steady-state levels
    const BlockLevels lv = block_levels(r.prof, false);
    AppNode f1{.kind = LayerKind::kLinearProjection, .name = "ffn.ffn1", .tokens = tokens, .in_dim = 768,
               .out_dim = 3072, .entry_level = lv.ffn1, .depth_cost = 1,
               .aggregation = AggregationAxis::kEmbeddingWise, .calibration_row = "ffn1"};
    const uint32_t a = app.add(f1);
    AppNode g{.kind = LayerKind::kGelu, .name = "ffn.gelu", .tokens = tokens, .in_dim = 3072, .out_dim = 3072,
              .entry_level = lv.gelu, .depth_cost = r.cfg.gelu_depth, .inputs = {a}, .calibration_row = "gelu"};
    const uint32_t b = app.add(g);
    AppNode f2{.kind = LayerKind::kLinearProjection, .name = "ffn.ffn2", .tokens = tokens, .in_dim = 3072,
               .out_dim = 768, .entry_level = lv.ffn2, .depth_cost = 1,
               .aggregation = AggregationAxis::kEmbeddingWise, .inputs = {b}, .calibration_row = "ffn2"};
    app.add(f2);
  }
  detail::AppLowering lw(app, r.prof, r.lay, LoweringOptions{});
  lw.g_.bundles.reserve(1u << 22);
  lw.g_.ops.reserve(1u << 22);
  r.he = lw.run();
  return r;
}

std::string slurp(const std::string& path) {
  std::ifstream f(path);
  std::stringstream s;
  s << f.rdbuf();
  return s.str();
}

int plan(const std::string& dir) {
  int bad = 0;
  struct Case { uint32_t n; uint64_t tokens; int kind; const char* name; };
  for (const Case& c : {Case{1u << 16, 128, 1, "ffn_n16_t128"}, Case{1u << 11, 32, 0, "block_n11_t32"}}) {
    Lowered r = lower(c.n, c.tokens, c.kind);
    aegis_compat::GraphArrays a = aegis_compat::to_arrays(r.he, r.prof, r.lay, r.cfg, c.tokens, (uint32_t)c.kind);
    aegis_graph* ingested = aegis_compat::ingest(a);
    const aegis_params ap = aegis_compat::params_of(r.prof);
    aegis_model m{(uint32_t)c.kind, 1, 768, 3072, 64, 64, c.tokens};
    aegis_graph* own = nullptr;
    aegis_compat::check(aegis_graph_build_params(&ap, &m, &own), nullptr);
    const std::string pa = dir + "/" + c.name + ".ingested.heops", pb = dir + "/" + c.name + ".own.heops";
    aegis_compat::check(aegis_graph_dump(ingested, pa.c_str()), nullptr);
    aegis_compat::check(aegis_graph_dump(own, pb.c_str()), nullptr);
    const bool same = slurp(pa) == slurp(pb);
    std::printf("%s: %zu ops, ingested %s own lowering\n", c.name, r.he.ops.size(), same ? "==" : "!=");
    bad += !same;
    aegis_graph_free(ingested);
    aegis_graph_free(own);
  }
  // a malformed graph is rejected with the reference's exception type
  Lowered r = lower(1u << 16, 128, 1);
  r.he.ops[3].out.lane_count = 1u << 20;
  try {
    aegis_graph_free(aegis_compat::ingest(aegis_compat::to_arrays(r.he, r.prof, r.lay, r.cfg, 128, 1)));
    std::printf("malformed graph accepted\n");
    ++bad;
  } catch (const std::invalid_argument& e) {
    std::printf("malformed graph rejected: %s\n", e.what());
  }
  return bad;
}

int run() {
  Lowered r = lower(1u << 10, 8, 1);
  aegis_compat::Executor ex(r.prof, 0);
  const std::vector<uint64_t> h = ex.exec_sequential(r.he, r.prof, r.lay, r.cfg, 8, 1);
  for (uint64_t v : h) std::printf("%016llx\n", (unsigned long long)v);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc >= 3 && !std::strcmp(argv[1], "plan")) return plan(argv[2]);
    if (argc >= 2 && !std::strcmp(argv[1], "run")) return run();
  } catch (const std::exception& e) {
    std::fprintf(stderr, "compat_test: %s\n", e.what());
    return 2;
  }
  std::fprintf(stderr, "usage: compat_test plan <dir> | run\n");
  return 2;
}

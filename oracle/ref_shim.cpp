// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// Thin extern "C" shim over the UNMODIFIED reference headers under
// /root/reference/proj/include (compiled in place by oracle/Makefile, output
// only into oracle/_ref/).  It exposes exactly the reference pieces that
// compile as shipped (SURVEY.md §0 build-status table):
//   rns_math.hpp  NegacyclicNtt (rns_math.hpp:44-123), negacyclic_automorphism
//                 (:127-139), rotation_galois_power (:142-149), CrtBasis
//                 (:153-193), div_round (:196-202)
//   ckks.hpp / graph.hpp / he_ir.hpp  build_transformer_graph (graph.hpp:168)
//                 and lower_app_to_he (he_ir.hpp:683) -> golden HE-op graphs.
// poly_ir.hpp / placement.hpp / comm_plan.hpp do not compile unmodified
// (poly_ir.hpp:335,:339; comm_plan.hpp:529) and are not used.
//
// he_ir.hpp holds `const CtBundle&` references across make_bundle() (e.g.
// he_ir.hpp:226->228), which dangles when g_.bundles reallocates.  We do not
// edit the header; instead the shim reaches the private lowering state and
// reserves the bundle vector before run(), so no reallocation (and no
// use-after-free) can happen.  The emitted graph is otherwise untouched.
#include <algorithm>
#include <array>
#include <cstdint>
#include <cstdio>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#define private public
#include "heplan/rns_math.hpp"
#include "heplan/ckks.hpp"
#include "heplan/graph.hpp"
#include "heplan/he_ir.hpp"
#undef private

using namespace heplan;

extern "C" {

// --- rns_math.hpp ---------------------------------------------------------
int ref_ntt(uint32_t n, uint64_t p, uint64_t* data, int inverse) {
  try {
    NegacyclicNtt ntt(n, p);
    std::vector<uint64_t> a(data, data + n);
    if (inverse) ntt.inverse(a); else ntt.forward(a);
    std::copy(a.begin(), a.end(), data);
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_ntt: %s\n", e.what());
    return -1;
  }
}

// Batched variant for timing the reference NTT as the CPU baseline: one
// NegacyclicNtt per prime, `count` limbs of n coefficients, limb i uses
// primes[i % nprimes].  Tables are built outside the timed call.
struct RefNttSet { std::vector<std::unique_ptr<NegacyclicNtt>> t; };
void* ref_ntt_set_create(uint32_t n, const uint64_t* primes, uint32_t nprimes) {
  auto* s = new RefNttSet;
  for (uint32_t i = 0; i < nprimes; ++i) s->t.emplace_back(new NegacyclicNtt(n, primes[i]));
  return s;
}
void ref_ntt_set_destroy(void* s) { delete static_cast<RefNttSet*>(s); }
int ref_ntt_set_run(void* sp, uint64_t* data, uint32_t count, int inverse, int threads) {
  auto* s = static_cast<RefNttSet*>(sp);
  const uint32_t n = s->t[0]->degree();
  #pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
  for (long i = 0; i < (long)count; ++i) {
    const NegacyclicNtt& t = *s->t[i % s->t.size()];
    std::vector<uint64_t> a(data + (size_t)i * n, data + (size_t)(i + 1) * n);
    if (inverse) t.inverse(a); else t.forward(a);
    std::copy(a.begin(), a.end(), data + (size_t)i * n);
  }
  return 0;
}

int ref_automorphism(uint32_t n, uint64_t k, uint64_t p, const uint64_t* in, uint64_t* out) {
  std::vector<uint64_t> a(in, in + n);
  std::vector<uint64_t> r = negacyclic_automorphism(a, k, p);
  std::copy(r.begin(), r.end(), out);
  return 0;
}

uint64_t ref_galois(int offset, uint32_t degree) { return rotation_galois_power(offset, degree); }

// Centered CRT lift of one residue vector (toy bases only: prod(p) < 2^127).
// Returns the value as two's-complement 128-bit in (lo, hi).
int ref_lift_centered(const uint64_t* primes, uint32_t k, const uint64_t* residues,
                      uint64_t* lo, int64_t* hi) {
  try {
    CrtBasis b(std::vector<uint64_t>(primes, primes + k));
    i128 v = b.lift_centered(std::vector<uint64_t>(residues, residues + k));
    *lo = (uint64_t)(u128)v;
    *hi = (int64_t)(v >> 64);
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_lift_centered: %s\n", e.what());
    return -1;
  }
}

uint64_t ref_crt_reduce(uint64_t lo, int64_t hi, uint64_t p) {
  i128 v = ((i128)hi << 64) | (i128)lo;
  return CrtBasis::reduce(v, p);
}

void ref_div_round(uint64_t nlo, int64_t nhi, uint64_t dlo, int64_t dhi, uint64_t* qlo, int64_t* qhi) {
  i128 n = ((i128)nhi << 64) | (i128)nlo;
  i128 d = ((i128)dhi << 64) | (i128)dlo;
  i128 q = div_round(n, d);
  *qlo = (uint64_t)(u128)q;
  *qhi = (int64_t)(q >> 64);
}

// --- ckks.hpp KATs ----------------------------------------------------------
uint64_t ref_ciphertext_bytes(uint32_t n, uint32_t level, uint32_t comps) {
  CkksProfile p{n, n / 2, 35, 4, 8, 14};
  return ciphertext_bytes(p, level, comps);
}
uint64_t ref_key_switch_key_bytes(uint32_t n, uint32_t chain, uint32_t special) {
  CkksProfile p{n, n / 2, chain, special, 8, 14};
  return key_switch_key_bytes(p);
}

// --- he_ir.hpp: dump the golden HE-op graph ----------------------------------
// kind: 0 = transformer (layers blocks), 1 = FFN only at steady-state levels
// (ffn1 @17 -> gelu @16 -> ffn2 @2).
int ref_dump_he(uint32_t n, uint32_t chain, uint32_t special, uint32_t lboot,
                uint32_t s_tok, uint32_t model_dim, uint32_t head_dim, uint32_t ffn_dim,
                uint64_t tokens, uint32_t layers, int kind, int exact, const char* path) {
  try {
    CkksProfile prof{n, n / 2, chain, special, 8, lboot};
    prof.validate();
    PackingLayout lay{s_tok, model_dim, head_dim};
    lay.validate(prof);
    TransformerConfig cfg;
    cfg.layer_count = layers;
    cfg.model_dim = model_dim;
    cfg.ffn_dim = ffn_dim;
    AppGraph app;
    if (kind == 0) {
      app = build_transformer_graph(cfg, prof, tokens);
    } else {
      const BlockLevels lv = block_levels(prof, false);
      AppNode f1{.kind = LayerKind::kLinearProjection, .name = "ffn.ffn1", .tokens = tokens,
                 .in_dim = model_dim, .out_dim = ffn_dim, .entry_level = lv.ffn1,
                 .depth_cost = 1, .aggregation = AggregationAxis::kEmbeddingWise,
                 .calibration_row = "ffn1"};
      const uint32_t a = app.add(f1);
      AppNode g{.kind = LayerKind::kGelu, .name = "ffn.gelu", .tokens = tokens,
                .in_dim = ffn_dim, .out_dim = ffn_dim, .entry_level = lv.gelu,
                .depth_cost = cfg.gelu_depth, .inputs = {a}, .calibration_row = "gelu"};
      const uint32_t b = app.add(g);
      AppNode f2{.kind = LayerKind::kLinearProjection, .name = "ffn.ffn2", .tokens = tokens,
                 .in_dim = ffn_dim, .out_dim = model_dim, .entry_level = lv.ffn2,
                 .depth_cost = 1, .aggregation = AggregationAxis::kEmbeddingWise,
                 .inputs = {b}, .calibration_row = "ffn2"};
      app.add(f2);
    }
    LoweringOptions opts;
    opts.exact = exact != 0;
    detail::AppLowering lw(app, prof, lay, opts);
    lw.g_.bundles.reserve(1u << 22);  // see header comment: avoids the he_ir.hpp UAF
    lw.g_.ops.reserve(1u << 22);
    HeOpGraph he = lw.run();

    FILE* f = std::fopen(path, "w");
    if (!f) return -2;
    std::fprintf(f, "# heops v1 N=%u L=%u K=%u lboot=%u stok=%u d=%u hd=%u dff=%u T=%llu layers=%u kind=%d exact=%d\n",
                 n, chain, special, lboot, s_tok, model_dim, head_dim, ffn_dim,
                 (unsigned long long)tokens, layers, kind, exact);
    std::fprintf(f, "inputs");
    for (uint32_t b : he.graph_inputs) std::fprintf(f, " %u", b);
    std::fprintf(f, "\n");
    for (const CtBundle& b : he.bundles)
      std::fprintf(f, "B %u %u %u %u %u %u %u %u %s\n", b.id, b.lanes, b.level, b.components,
                   (unsigned)b.cls, b.chunk_period, (unsigned)b.replicate_hint, b.app_node,
                   b.tag.c_str());
    for (const HeOp& o : he.ops) {
      std::fprintf(f, "O %u %u %d %u %u %u %d %d %d %llu %u %u %u %zu", o.id, (unsigned)o.kind,
                   o.rot_offset, o.out.bundle, o.out.lane, o.out.lane_count, (int)o.accumulate,
                   (int)o.aligned, o.phase, (unsigned long long)o.work, o.use_level, o.app_node,
                   (unsigned)o.aggregation, o.ins.size());
      for (const LaneSlice& s : o.ins) std::fprintf(f, " %u %u %u", s.bundle, s.lane, s.lane_count);
      std::fprintf(f, "\n");
    }
    std::fclose(f);
    return (int)he.ops.size();
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_dump_he: %s\n", e.what());
    return -1;
  }
}

}  // extern "C"

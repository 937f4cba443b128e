// heplan_compat.hpp -- the C++ binding a heplan caller includes to run its
// HE-op graphs on libaegis.  Header-only; needs the
// reference headers (heplan/he_ir.hpp) on the include path and links
// libaegis.so.  Nothing of libaegis itself includes this file: the product is
// the C-ABI in include/aegis.h, this is the reference-side adapter over it.
//
//   * check()          AEGIS_E* codes -> the reference's exception types
//                      (std::invalid_argument ckks.hpp:149 / graph.hpp:100,
//                      std::logic_error he_ir.hpp:191, std::runtime_error).
//   * params_of()      CkksProfile (ckks.hpp:21-46) -> aegis_params.
//   * to_arrays()      an in-memory heplan::HeOpGraph (he_ir.hpp:101-120) ->
//                      the aegis_graph_from_ops descriptors, field for field.
//   * Executor         exec_sequential on one GPU: ingest
//                      the caller's HeOpGraph (no text round trip), generate
//                      the keys it names (poly_ir.hpp:300-305), run it, and
//                      return the per-bundle content hashes.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "heplan/he_ir.hpp"
#include "../../include/aegis.h"

namespace aegis_compat {

inline void check(int rc, const aegis_ctx* c) {
  if (rc == AEGIS_OK) return;
  const std::string m = aegis_last_error(c) ? aegis_last_error(c) : "aegis error";
  if (rc == AEGIS_EINVAL) throw std::invalid_argument(m);
  if (rc == AEGIS_ELOGIC) throw std::logic_error(m);
  throw std::runtime_error(m);
}

inline uint32_t log2_exact(uint32_t n) {
  uint32_t l = 0;
  while ((1u << l) < n) ++l;
  if ((1u << l) != n) throw std::invalid_argument("ring_degree must be a power of two");
  return l;
}

// seeds of the synthetic workload
inline aegis_params params_of(const heplan::CkksProfile& p, uint64_t seed_input = 0xAE615,
                              uint64_t seed_weight = 0xAE616, uint64_t seed_key = 0xAE617) {
  return aegis_params{log2_exact(p.ring_degree), p.chain_length, p.special_prime_count, p.bootstrap_level,
                      seed_input, seed_weight, seed_key};
}

struct GraphArrays {
  aegis_graph_meta meta{};
  std::vector<aegis_bundle_desc> bundles;
  std::vector<aegis_op_desc> ops;
  std::vector<uint32_t> inputs;
};

// kind: 0 = transformer blocks (build_transformer_graph), 1 = FFN only
inline GraphArrays to_arrays(const heplan::HeOpGraph& g, const heplan::CkksProfile& p,
                             const heplan::PackingLayout& lay, const heplan::TransformerConfig& cfg,
                             uint64_t tokens, uint32_t kind) {
  GraphArrays a;
  a.meta = aegis_graph_meta{log2_exact(p.ring_degree), p.chain_length, p.bootstrap_level, lay.slots_per_token,
                            lay.model_dim, lay.head_dim, cfg.ffn_dim, cfg.layer_count, kind, tokens};
  a.bundles.reserve(g.bundles.size());
  for (const heplan::CtBundle& b : g.bundles)
    a.bundles.push_back(aegis_bundle_desc{b.lanes, b.level, b.components, (uint32_t)b.cls,
                                          (uint32_t)b.aggregation, b.app_node, b.chunk_period,
                                          (uint32_t)b.replicate_hint, b.tag.c_str()});
  a.ops.reserve(g.ops.size());
  for (const heplan::HeOp& op : g.ops) {
    if (op.ins.size() > AEGIS_MAX_OP_INPUTS)
      throw std::invalid_argument("HeOp " + std::to_string(op.id) + " has more operands than the executor takes");
    aegis_op_desc d{};
    d.kind = (uint32_t)op.kind;
    d.accumulate = op.accumulate;
    d.aligned = op.aligned;
    d.aggregation = (uint32_t)op.aggregation;
    d.rot_offset = op.rot_offset;
    d.phase = op.phase;
    d.out = aegis_slice{op.out.bundle, op.out.lane, op.out.lane_count};
    d.in_count = (uint32_t)op.ins.size();
    for (size_t k = 0; k < op.ins.size(); ++k)
      d.ins[k] = aegis_slice{op.ins[k].bundle, op.ins[k].lane, op.ins[k].lane_count};
    d.work = op.work;
    d.use_level = op.use_level;
    d.app_node = op.app_node;
    a.ops.push_back(d);
  }
  a.inputs = g.graph_inputs;
  return a;
}

// Plan-only ingest (no device): the graph the executor would run.
inline aegis_graph* ingest(const GraphArrays& a) {
  aegis_graph* out = nullptr;
  check(aegis_graph_from_ops(&a.meta, a.bundles.data(), (uint32_t)a.bundles.size(), a.ops.data(), a.ops.size(),
                             a.inputs.data(), (uint32_t)a.inputs.size(), &out),
        nullptr);
  return out;
}

class Executor {
 public:
  Executor(const heplan::CkksProfile& p, int device) {
    const aegis_params ap = params_of(p);
    check(aegis_ctx_create(&ap, device, &ctx_), nullptr);
  }
  ~Executor() { aegis_ctx_destroy(ctx_); }
  Executor(const Executor&) = delete;
  Executor& operator=(const Executor&) = delete;

  aegis_ctx* context() { return ctx_; }

  // exec_sequential over a caller-held HeOpGraph: returns
  // the DESIGN.md §2.4 hash of every bundle (0 = never materialised)
  std::vector<uint64_t> exec_sequential(const heplan::HeOpGraph& g, const heplan::CkksProfile& p,
                                        const heplan::PackingLayout& lay, const heplan::TransformerConfig& cfg,
                                        uint64_t tokens, uint32_t kind) {
    const GraphArrays a = to_arrays(g, p, lay, cfg, tokens, kind);
    aegis_graph* graph = ingest(a);
    std::vector<uint64_t> hashes(a.bundles.size());
    try {
      uint32_t nk = 0;
      check(aegis_graph_key_ids(graph, nullptr, 0, &nk), ctx_);
      std::vector<uint64_t> ids(nk);
      check(aegis_graph_key_ids(graph, ids.data(), nk, &nk), ctx_);
      check(aegis_keys_generate(ctx_, ids.data(), nk), ctx_);
      check(aegis_graph_run(ctx_, graph, -1, hashes.data(), hashes.size()), ctx_);
      check(aegis_sync(ctx_), ctx_);
    } catch (...) {
      aegis_graph_free(graph);
      throw;
    }
    aegis_graph_free(graph);
    return hashes;
  }

 private:
  aegis_ctx* ctx_ = nullptr;
};

}  // namespace aegis_compat

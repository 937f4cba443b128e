// heplan_ir.h -- the reference's operator API, restated for libaegis.
//
// These are the data types and "layer drivers" of the reference planner
// (graph.hpp, he_ir.hpp) that the hot path executes: an application graph of
// BERT layers (graph.hpp:63-121, 125-299) lowered to bundled HE operators
// (he_ir.hpp:57-120, 328-669).  Names, fields and emitted sequences match the
// reference one-for-one so that a heplan caller can hand its HeOpGraph to the
// GPU executor unchanged; tests/test_lowering.py checks the emitted graphs
// against golden dumps produced by the unmodified reference (oracle/_ref).
// Only bundled lowering is provided (LoweringOptions::exact is the verifier's
// toy mode, he_ir.hpp:122-125, and is out of scope -- DESIGN.md §5).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace aegis::heplan {

struct CkksProfile {  // ckks.hpp:21-46
  uint32_t ring_degree = 0, slot_count = 0, chain_length = 0, special_prime_count = 0;
  uint32_t bytes_per_coefficient = 8, bootstrap_level = 0;
  uint32_t post_boot_level() const { return chain_length - bootstrap_level; }
};
struct PackingLayout {  // ckks.hpp:50-72
  uint32_t slots_per_token = 0, model_dim = 0, head_dim = 0;
};

enum class LayerKind : uint8_t {  // graph.hpp:19-29
  kLinearProjection, kAttentionScore, kSoftmax, kAttentionOutput, kOutputProjection,
  kLayerNorm, kGelu, kBootstrapping, kResidual,
};
enum class AggregationAxis : uint8_t { kNone, kTokenWise, kEmbeddingWise, kHeadWise };

struct AppNode {  // graph.hpp:63-77
  uint32_t id = 0;
  LayerKind kind = LayerKind::kLinearProjection;
  std::string name;
  uint64_t tokens = 0;
  uint32_t in_dim = 0, out_dim = 0, entry_level = 0, depth_cost = 0;
  AggregationAxis aggregation = AggregationAxis::kNone;
  std::vector<uint32_t> inputs;
  uint32_t block = 0, sub_tensors = 1;
};
struct AppGraph {
  std::vector<AppNode> nodes;
  uint32_t add(AppNode n);
  void validate(const CkksProfile& p) const;  // graph.hpp:95-115
};

struct TransformerConfig {  // graph.hpp:125-137
  uint32_t layer_count = 12, model_dim = 768, ffn_dim = 3072, head_count = 12;
  uint32_t softmax_depth = 16, softmax_pre_depth = 3, gelu_depth = 14, layernorm_depth = 16;
};

AppGraph build_transformer_graph(const TransformerConfig& cfg, const CkksProfile& p, uint64_t tokens);
// ffn1 -> gelu -> ffn2 at steady-state levels
AppGraph build_ffn_graph(const TransformerConfig& cfg, const CkksProfile& p, uint64_t tokens);

enum class HeOpKind : uint8_t { kEncode, kPAdd, kCAdd, kPMult, kCMult, kRot, kRelin, kRescale, kBoot };
enum class BundleClass : uint8_t { kInput, kActivation, kRotated, kWeight, kScore };

struct CtBundle {  // he_ir.hpp:57-74
  uint32_t id = 0, lanes = 1, level = 0, components = 2;
  BundleClass cls = BundleClass::kActivation;
  AggregationAxis aggregation = AggregationAxis::kNone;
  uint32_t token_begin = 0, token_end = 0;
  uint32_t app_node = 0, chunk_period = 0;
  bool replicate_hint = false;
  std::string tag;
};
struct LaneSlice {
  uint32_t bundle = 0, lane = 0, lane_count = 1;
};
struct HeOp {  // he_ir.hpp:84-99
  uint32_t id = 0;
  HeOpKind kind = HeOpKind::kCAdd;
  int rot_offset = 0;
  LaneSlice out{};
  std::vector<LaneSlice> ins;
  bool accumulate = false, aligned = false;
  int phase = -1;
  uint64_t work = 0;
  uint32_t use_level = 0, app_node = 0;
  AggregationAxis aggregation = AggregationAxis::kNone;
  uint64_t lane_ops() const { return work ? work : out.lane_count; }
};
struct HeOpGraph {
  std::vector<CtBundle> bundles;
  std::vector<HeOp> ops;
  std::vector<uint32_t> graph_inputs;
};

// he_ir.hpp:683-687 (bundled mode)
HeOpGraph lower_app_to_he(const AppGraph& app, const CkksProfile& p, const PackingLayout& layout);

// text round trip in the tests/golden heops format
std::string dump_heops(const HeOpGraph& g, const std::string& header);
HeOpGraph parse_heops(const std::string& text);
void validate_heops(const HeOpGraph& g);  // throws std::invalid_argument

}  // namespace aegis::heplan

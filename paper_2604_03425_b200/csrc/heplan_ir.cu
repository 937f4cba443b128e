// heplan_ir.cu -- layer drivers: BERT application graph and its bundled
// HE-operator lowering (restating graph.hpp:147-299 and he_ir.hpp:143-669).
//
// The emitted HeOpGraph must be identical -- bundle ids, tags, op order and
// every field -- to the reference's lower_app_to_he in bundled mode, because
// bundle ids seed the kGenerate weights and the executor replays the op list
// verbatim.  tests/test_lowering.py diffs our dump against golden dumps made
// by the unmodified reference (tests/golden/*.heops.gz).
#include <sstream>
#include <stdexcept>

#include "heplan_ir.h"

namespace aegis::heplan {

uint32_t AppGraph::add(AppNode n) {
  n.id = static_cast<uint32_t>(nodes.size());
  for (uint32_t in : n.inputs)
    if (in >= n.id) throw std::invalid_argument("app graph input out of order");
  nodes.push_back(std::move(n));
  return nodes.back().id;
}

namespace {
uint32_t exit_level(const AppNode& n, const CkksProfile& p) {  // graph.hpp:117-120
  return n.kind == LayerKind::kBootstrapping ? p.post_boot_level() : n.entry_level - n.depth_cost;
}
}  // namespace

void AppGraph::validate(const CkksProfile& p) const {
  for (const AppNode& n : nodes) {
    if (n.entry_level == 0 || n.entry_level > p.chain_length)
      throw std::invalid_argument("node " + n.name + ": entry level out of range");
    if (n.kind != LayerKind::kBootstrapping && n.entry_level < n.depth_cost + 1)
      throw std::invalid_argument("level underflow at node " + n.name + ": entry " +
                                  std::to_string(n.entry_level) + " cannot pay depth " +
                                  std::to_string(n.depth_cost));
    for (uint32_t in : n.inputs) {
      const AppNode& src = nodes.at(in);
      const uint32_t avail = exit_level(src, p);
      if (avail < n.entry_level)
        throw std::invalid_argument("level underflow at node " + n.name + ": needs " +
                                    std::to_string(n.entry_level) + " but " + src.name + " exits at " +
                                    std::to_string(avail));
    }
  }
}

namespace {

struct Levels {  // graph.hpp:142-163
  uint32_t qkv, score, softmax, att_out, out_proj, layer_norm, ffn1, gelu, ffn2;
};
Levels schedule(const CkksProfile& p, bool first) {
  const uint32_t steady = p.post_boot_level();
  if (steady < 21) throw std::invalid_argument("transformer schedule needs a usable depth of 21");
  const uint32_t top = first ? p.chain_length : steady;
  return Levels{top, top - 1, top - 2, top - 18, steady - 19, steady - 4, steady - 4, steady - 5, steady - 19};
}

AppNode node(LayerKind k, const std::string& name, uint64_t tokens, uint32_t in_dim, uint32_t out_dim,
             uint32_t entry, uint32_t depth, AggregationAxis agg, std::vector<uint32_t> inputs, uint32_t block,
             uint32_t sub = 1) {
  AppNode n;
  n.kind = k;
  n.name = name;
  n.tokens = tokens;
  n.in_dim = in_dim;
  n.out_dim = out_dim;
  n.entry_level = entry;
  n.depth_cost = depth;
  n.aggregation = agg;
  n.inputs = std::move(inputs);
  n.block = block;
  n.sub_tensors = sub;
  return n;
}

}  // namespace

AppGraph build_transformer_graph(const TransformerConfig& cfg, const CkksProfile& p, uint64_t T) {
  using LK = LayerKind;
  using AX = AggregationAxis;
  AppGraph g;
  const uint32_t d = cfg.model_dim;
  bool chained = false;
  uint32_t carry = 0;  // output of the previous block
  for (uint32_t b = 0; b < cfg.layer_count; ++b) {
    const Levels lv = schedule(p, b == 0);
    const std::string pfx = "block" + std::to_string(b) + ".";
    const std::vector<uint32_t> from_prev = chained ? std::vector<uint32_t>{carry} : std::vector<uint32_t>{};
    const uint32_t skip = chained ? carry : 0;
    const uint32_t qkv = g.add(node(LK::kLinearProjection, pfx + "qkv", T, d, 3 * d, lv.qkv, 1, AX::kEmbeddingWise,
                                    from_prev, b, 3));
    const uint32_t sc = g.add(node(LK::kAttentionScore, pfx + "score", T, d, d, lv.score, 1, AX::kHeadWise, {qkv}, b));
    const uint32_t sm = g.add(node(LK::kSoftmax, pfx + "softmax", T, d, d, lv.softmax, cfg.softmax_depth,
                                   AX::kTokenWise, {sc}, b));
    const uint32_t av = g.add(node(LK::kAttentionOutput, pfx + "att_out", T, d, d, lv.att_out, 1, AX::kHeadWise,
                                   {qkv, sm}, b));
    const uint32_t wo = g.add(node(LK::kOutputProjection, pfx + "out_proj", T, d, d, lv.out_proj, 1,
                                   AX::kEmbeddingWise, {av}, b));
    const uint32_t r1 = g.add(node(LK::kResidual, pfx + "residual_att", T, d, d, lv.out_proj - 1, 0, AX::kNone,
                                   chained ? std::vector<uint32_t>{wo, skip} : std::vector<uint32_t>{wo}, b));
    const uint32_t b1 = g.add(node(LK::kBootstrapping, pfx + "boot_att", T, d, d, lv.out_proj - 1, 0, AX::kNone,
                                   {r1}, b));
    const uint32_t ln1 = g.add(node(LK::kLayerNorm, pfx + "layer_norm_post", T, d, d, lv.layer_norm,
                                    cfg.layernorm_depth, AX::kTokenWise, {b1}, b));
    const uint32_t b2 = g.add(node(LK::kBootstrapping, pfx + "boot_ln_post", T, d, d,
                                   lv.layer_norm - cfg.layernorm_depth, 0, AX::kNone, {ln1}, b));
    const uint32_t f1 = g.add(node(LK::kLinearProjection, pfx + "ffn1", T, d, cfg.ffn_dim, lv.ffn1, 1,
                                   AX::kEmbeddingWise, {b2}, b));
    const uint32_t ge = g.add(node(LK::kGelu, pfx + "gelu", T, cfg.ffn_dim, cfg.ffn_dim, lv.gelu, cfg.gelu_depth,
                                   AX::kNone, {f1}, b));
    const uint32_t f2 = g.add(node(LK::kLinearProjection, pfx + "ffn2", T, cfg.ffn_dim, d, lv.ffn2, 1,
                                   AX::kEmbeddingWise, {ge}, b));
    const uint32_t r2 = g.add(node(LK::kResidual, pfx + "residual_ffn", T, d, d, lv.ffn2 - 1, 0, AX::kNone,
                                   {f2, b1}, b));
    const uint32_t b3 = g.add(node(LK::kBootstrapping, pfx + "boot_ffn", T, d, d, lv.ffn2 - 1, 0, AX::kNone, {r2}, b));
    const uint32_t ln2 = g.add(node(LK::kLayerNorm, pfx + "layer_norm_pre", T, d, d, lv.layer_norm,
                                    cfg.layernorm_depth, AX::kTokenWise, {b3}, b));
    carry = g.add(node(LK::kBootstrapping, pfx + "boot_ln_pre", T, d, d, lv.layer_norm - cfg.layernorm_depth, 0,
                       AX::kNone, {ln2}, b));
    chained = true;
  }
  return g;
}

AppGraph build_ffn_graph(const TransformerConfig& cfg, const CkksProfile& p, uint64_t T) {
  const Levels lv = schedule(p, false);
  AppGraph g;
  const uint32_t f1 = g.add(node(LayerKind::kLinearProjection, "ffn.ffn1", T, cfg.model_dim, cfg.ffn_dim, lv.ffn1, 1,
                                 AggregationAxis::kEmbeddingWise, {}, 0));
  const uint32_t ge = g.add(node(LayerKind::kGelu, "ffn.gelu", T, cfg.ffn_dim, cfg.ffn_dim, lv.gelu, cfg.gelu_depth,
                                 AggregationAxis::kNone, {f1}, 0));
  g.add(node(LayerKind::kLinearProjection, "ffn.ffn2", T, cfg.ffn_dim, cfg.model_dim, lv.ffn2, 1,
             AggregationAxis::kEmbeddingWise, {ge}, 0));
  return g;
}

// ---------------------------------------------------------------------------
// Bundled lowering (he_ir.hpp:143-669).
// ---------------------------------------------------------------------------
namespace {

class Lowerer {
 public:
  Lowerer(const AppGraph& app, const CkksProfile& p, const PackingLayout& lay) : app_(app), p_(p), lay_(lay) {
    app_.validate(p_);
  }

  HeOpGraph run() {
    produced_.assign(app_.nodes.size(), kNone);
    for (const AppNode& n : app_.nodes) produced_[n.id] = lower(n);
    return std::move(g_);
  }

 private:
  static constexpr uint32_t kNone = 0xffffffffu;

  uint32_t tokens_per_ct() const { return p_.slot_count / lay_.slots_per_token; }
  uint32_t groups(uint64_t T) const { return (uint32_t)((T + tokens_per_ct() - 1) / tokens_per_ct()); }
  uint32_t lanes_for(uint64_t T, uint32_t dim) const {
    return groups(T) * ((dim + lay_.slots_per_token - 1) / lay_.slots_per_token);
  }
  uint32_t ladder_steps() const {  // ceil(log2 s_tok), at least 1 (he_ir.hpp:497-498)
    uint32_t s = 1;
    while ((1u << s) < lay_.slots_per_token) ++s;
    return s;
  }
  const CtBundle& B(uint32_t id) const { return g_.bundles[id]; }

  uint32_t fresh(const AppNode& n, uint32_t lanes, uint32_t level, uint32_t comps, BundleClass cls,
                 const std::string& suffix) {
    CtBundle b;
    b.id = (uint32_t)g_.bundles.size();
    b.lanes = lanes;
    b.level = level;
    b.components = comps;
    b.cls = cls;
    b.aggregation = n.aggregation;
    b.token_begin = 0;
    b.token_end = (uint32_t)n.tokens;
    b.app_node = n.id;
    b.replicate_hint = replicate_;
    b.tag = n.name + suffix;
    g_.bundles.push_back(std::move(b));
    return g_.bundles.back().id;
  }

  uint32_t source(const AppNode& n, size_t idx = 0) {
    if (n.inputs.empty()) {  // fresh client activations at the entry level
      const uint32_t b = fresh(n, lanes_for(n.tokens, n.in_dim), n.entry_level, 2, BundleClass::kInput, ".in");
      g_.bundles[b].aggregation = AggregationAxis::kNone;
      g_.graph_inputs.push_back(b);
      return b;
    }
    const uint32_t out = produced_[n.inputs.at(idx)];
    if (out == kNone) throw std::logic_error("app node consumed before being lowered");
    return out;
  }

  void push(HeOp op, const AppNode& n) {
    op.app_node = n.id;
    if (op.aggregation == AggregationAxis::kNone) op.aggregation = n.aggregation;
    op.id = (uint32_t)g_.ops.size();
    g_.ops.push_back(std::move(op));
  }

  static HeOp make(HeOpKind k, LaneSlice out, std::vector<LaneSlice> ins, uint32_t use_level, int phase = -1) {
    HeOp op;
    op.kind = k;
    op.out = out;
    op.ins = std::move(ins);
    op.use_level = use_level;
    op.phase = phase;
    return op;
  }
  LaneSlice all(uint32_t b) const { return LaneSlice{b, 0, B(b).lanes}; }

  uint32_t rotate(const AppNode& n, uint32_t src, int off, uint32_t level, int phase = -1) {
    const uint32_t lanes = B(src).lanes, period = B(src).chunk_period;
    const bool rep = B(src).replicate_hint;
    const uint32_t r = fresh(n, lanes, level, 2, BundleClass::kRotated, ".rot" + std::to_string(off));
    g_.bundles[r].chunk_period = period;
    g_.bundles[r].replicate_hint = rep;
    HeOp op = make(HeOpKind::kRot, LaneSlice{r, 0, lanes}, {LaneSlice{src, 0, lanes}}, level, phase);
    op.rot_offset = off;
    push(op, n);
    return r;
  }

  uint32_t relinearize(const AppNode& n, uint32_t b) {
    g_.bundles[b].components = 2;
    push(make(HeOpKind::kRelin, all(b), {all(b)}, B(b).level), n);
    return b;
  }

  uint32_t rescale(const AppNode& n, uint32_t b) {
    const uint32_t level = B(b).level, lanes = B(b).lanes, comps = B(b).components;
    const BundleClass cls = B(b).cls;
    if (level < 2) throw std::invalid_argument("level underflow at node " + n.name + ": cannot rescale below level 1");
    const uint32_t out = fresh(n, lanes, level - 1, comps, cls, ".rs");
    g_.bundles[out].cls = cls == BundleClass::kScore ? BundleClass::kScore : BundleClass::kActivation;
    push(make(HeOpKind::kRescale, LaneSlice{out, 0, lanes}, {LaneSlice{b, 0, lanes}}, level), n);
    return out;
  }

  // depth successive squarings: CMult(x, x) -> Relin -> Rescale (he_ir.hpp:305-322)
  uint32_t squarings(const AppNode& n, uint32_t src, uint32_t depth, const std::string& what) {
    uint32_t cur = src;
    for (uint32_t i = 0; i < depth; ++i) {
      const uint32_t lanes = B(cur).lanes, level = B(cur).level;
      const uint32_t sq = fresh(n, lanes, level, 3, B(cur).cls, "." + what + std::to_string(i));
      push(make(HeOpKind::kCMult, LaneSlice{sq, 0, lanes}, {LaneSlice{cur, 0, lanes}, LaneSlice{cur, 0, lanes}},
                level),
           n);
      relinearize(n, sq);
      cur = rescale(n, sq);
    }
    return cur;
  }

  // relinearised CMult of a[a_lane, a_lane+count) with b (he_ir.hpp:400-424)
  uint32_t product(const AppNode& n, uint32_t a, uint32_t a_lane, uint32_t count, uint32_t b, int phase,
                   const std::string& suffix) {
    const uint32_t prod = fresh(n, count, n.entry_level, 3, BundleClass::kActivation, suffix);
    HeOp mul = make(HeOpKind::kCMult, LaneSlice{prod, 0, count},
                    {LaneSlice{a, a_lane, count}, LaneSlice{b, 0, std::min(B(b).lanes, count)}}, n.entry_level, phase);
    mul.aligned = true;
    push(mul, n);
    HeOp rl = make(HeOpKind::kRelin, LaneSlice{prod, 0, count}, {LaneSlice{prod, 0, count}}, n.entry_level, phase);
    g_.bundles[prod].components = 2;
    push(rl, n);
    return prod;
  }

  void accumulate(const AppNode& n, uint32_t acc, uint32_t src, int phase, bool aligned, uint64_t work) {
    HeOp op = make(HeOpKind::kCAdd, all(acc), {all(src)}, B(acc).level, phase);
    if (aligned) op.ins[0].lane_count = B(acc).lanes;
    op.accumulate = true;
    op.aligned = aligned;
    op.work = work;
    push(op, n);
  }

  // --- layers ----------------------------------------------------------------
  uint32_t matmul(const AppNode& n) {  // he_ir.hpp:328-373 (bundled branch)
    const uint32_t src = source(n);
    const uint32_t in_l = lanes_for(n.tokens, n.in_dim), out_l = lanes_for(n.tokens, n.out_dim);
    const uint32_t tg = groups(n.tokens);
    const uint32_t c_in = in_l / tg, c_out = out_l / tg;
    const uint32_t acc = fresh(n, out_l, n.entry_level, 2, BundleClass::kActivation, ".acc");
    g_.bundles[acc].chunk_period = out_l / n.sub_tensors;
    for (uint32_t r = 0; r < lay_.slots_per_token; ++r) {
      const uint32_t x = r == 0 ? src : rotate(n, src, (int)r, n.entry_level, (int)r);
      const uint32_t w = fresh(n, c_in * c_out, n.entry_level, 1, BundleClass::kWeight, ".w" + std::to_string(r));
      push(make(HeOpKind::kEncode, LaneSlice{w, 0, c_in * c_out}, {}, 0), n);
      HeOp mac = make(HeOpKind::kPMult, all(acc), {all(x), all(w)}, B(acc).level, (int)r);
      mac.accumulate = true;
      mac.work = (uint64_t)in_l * c_out;
      push(mac, n);
    }
    return rescale(n, acc);
  }

  uint32_t scores(const AppNode& n) {  // he_ir.hpp:454-475
    const uint32_t qkv = source(n);
    const uint32_t heads = std::max<uint32_t>(1, n.in_dim / lay_.head_dim);
    const uint64_t vals = n.tokens * n.tokens * heads;
    const uint32_t s_lanes = (uint32_t)((vals + p_.slot_count - 1) / p_.slot_count);  // ckks.hpp:251-255
    const uint32_t q_lanes = std::max(1u, B(qkv).lanes / 3);
    const uint32_t acc = fresh(n, s_lanes, n.entry_level, 2, BundleClass::kScore, ".acc");
    for (uint32_t r = 0; r < lay_.head_dim; ++r) {
      const uint32_t x = r == 0 ? qkv : rotate(n, qkv, (int)r, n.entry_level, (int)r);
      const uint32_t prod = product(n, qkv, 0, q_lanes, x, (int)r, ".qk" + std::to_string(r));
      accumulate(n, acc, prod, (int)r, false, std::max(B(acc).lanes, B(prod).lanes));
    }
    return rescale(n, acc);
  }

  uint32_t softmax(const AppNode& n) {  // he_ir.hpp:477-519
    const uint32_t s = source(n);
    const uint32_t lanes = B(s).lanes;
    const uint32_t masked = fresh(n, lanes, B(s).level, 2, BundleClass::kScore, ".maxsub");
    push(make(HeOpKind::kCAdd, LaneSlice{masked, 0, lanes}, {LaneSlice{s, 0, lanes}, LaneSlice{s, 0, lanes}},
              B(s).level),
         n);
    uint32_t cur = squarings(n, masked, 1, "msub");
    const uint32_t pre = std::min<uint32_t>(3, n.depth_cost);
    cur = squarings(n, cur, pre - 1, "exp");
    for (uint32_t k = 0; k < ladder_steps(); ++k) {
      const uint32_t rot = rotate(n, cur, (int)(1u << k), B(cur).level);
      const uint32_t cl = B(cur).lanes;
      push(make(HeOpKind::kCAdd, LaneSlice{cur, 0, cl}, {LaneSlice{cur, 0, cl}, LaneSlice{rot, 0, cl}}, B(cur).level),
           n);
    }
    replicate_ = true;  // normalisation runs on the re-gathered scores
    cur = squarings(n, cur, n.depth_cost - pre, "norm");
    replicate_ = false;
    g_.bundles[cur].cls = BundleClass::kScore;
    return cur;
  }

  uint32_t attn_out(const AppNode& n) {  // he_ir.hpp:524-569
    const uint32_t v = source(n, 0), attn = source(n, 1);
    const uint32_t out_l = lanes_for(n.tokens, n.out_dim);
    const uint32_t v0 = (B(v).lanes / 3) * 2;
    const uint32_t acc = fresh(n, out_l, n.entry_level, 2, BundleClass::kActivation, ".acc");
    for (uint32_t r = 0; r < lay_.slots_per_token; ++r) {
      const uint32_t x = r == 0 ? attn : rotate(n, attn, (int)r, n.entry_level, (int)r);
      const uint32_t prod = product(n, v, v0, out_l, x, (int)r, ".av" + std::to_string(r));
      HeOp op = make(HeOpKind::kCAdd, LaneSlice{acc, 0, out_l}, {LaneSlice{prod, 0, out_l}}, n.entry_level, (int)r);
      op.accumulate = true;
      op.aligned = true;
      op.work = out_l;
      push(op, n);
    }
    return rescale(n, acc);
  }

  uint32_t layernorm(const AppNode& n) {  // he_ir.hpp:571-599
    const uint32_t src = source(n);
    const uint32_t lanes = B(src).lanes;
    const uint32_t sum = fresh(n, lanes, n.entry_level, 2, BundleClass::kActivation, ".sum");
    push(make(HeOpKind::kCAdd, LaneSlice{sum, 0, lanes}, {LaneSlice{src, 0, lanes}, LaneSlice{src, 0, lanes}},
              n.entry_level),
         n);
    for (uint32_t k = 0; k < ladder_steps(); ++k) {
      const uint32_t rot = rotate(n, sum, (int)(1u << k), n.entry_level);
      push(make(HeOpKind::kCAdd, LaneSlice{sum, 0, lanes}, {LaneSlice{sum, 0, lanes}, LaneSlice{rot, 0, lanes}},
                n.entry_level),
           n);
    }
    return squarings(n, sum, n.depth_cost, "ln");
  }

  uint32_t boot(const AppNode& n) {  // he_ir.hpp:601-613
    const uint32_t src = source(n);
    const uint32_t lanes = B(src).lanes;
    const uint32_t out = fresh(n, lanes, p_.post_boot_level(), 2, BundleClass::kActivation, ".boot");
    push(make(HeOpKind::kBoot, LaneSlice{out, 0, lanes}, {LaneSlice{src, 0, lanes}}, n.entry_level), n);
    return out;
  }

  uint32_t residual(const AppNode& n) {  // he_ir.hpp:615-628
    const uint32_t a = source(n, 0);
    const uint32_t b = n.inputs.size() > 1 ? source(n, 1) : a;
    const uint32_t lanes = B(a).lanes;
    const uint32_t out = fresh(n, lanes, n.entry_level, 2, BundleClass::kActivation, ".sum");
    push(make(HeOpKind::kCAdd, LaneSlice{out, 0, lanes},
              {LaneSlice{a, 0, lanes}, LaneSlice{b, 0, std::min(lanes, B(b).lanes)}}, n.entry_level),
         n);
    return out;
  }

  uint32_t lower(const AppNode& n) {
    switch (n.kind) {
      case LayerKind::kLinearProjection:
      case LayerKind::kOutputProjection: return matmul(n);
      case LayerKind::kAttentionScore: return scores(n);
      case LayerKind::kSoftmax: return softmax(n);
      case LayerKind::kAttentionOutput: return attn_out(n);
      case LayerKind::kLayerNorm: return layernorm(n);
      case LayerKind::kGelu: return squarings(n, source(n), n.depth_cost, "gelu");
      case LayerKind::kBootstrapping: return boot(n);
      case LayerKind::kResidual: return residual(n);
    }
    throw std::logic_error("unknown layer kind");
  }

  const AppGraph& app_;
  const CkksProfile& p_;
  const PackingLayout& lay_;
  HeOpGraph g_;
  std::vector<uint32_t> produced_;
  bool replicate_ = false;
};

}  // namespace

HeOpGraph lower_app_to_he(const AppGraph& app, const CkksProfile& p, const PackingLayout& layout) {
  return Lowerer(app, p, layout).run();
}

std::string dump_heops(const HeOpGraph& g, const std::string& header) {
  std::ostringstream o;
  o << header << "\n";
  o << "inputs";
  for (uint32_t b : g.graph_inputs) o << " " << b;
  o << "\n";
  for (const CtBundle& b : g.bundles)
    o << "B " << b.id << " " << b.lanes << " " << b.level << " " << b.components << " " << (unsigned)b.cls << " "
      << b.chunk_period << " " << (unsigned)b.replicate_hint << " " << b.app_node << " " << b.tag << "\n";
  for (const HeOp& op : g.ops) {
    o << "O " << op.id << " " << (unsigned)op.kind << " " << op.rot_offset << " " << op.out.bundle << " "
      << op.out.lane << " " << op.out.lane_count << " " << (int)op.accumulate << " " << (int)op.aligned << " "
      << op.phase << " " << op.work << " " << op.use_level << " " << op.app_node << " " << (unsigned)op.aggregation
      << " " << op.ins.size();
    for (const LaneSlice& s : op.ins) o << " " << s.bundle << " " << s.lane << " " << s.lane_count;
    o << "\n";
  }
  return o.str();
}

HeOpGraph parse_heops(const std::string& text) {
  HeOpGraph g;
  std::istringstream in(text);
  std::string line;
  while (std::getline(in, line)) {
    if (line.empty() || line[0] == '#') continue;
    std::istringstream s(line);
    std::string t;
    s >> t;
    if (t == "inputs") {
      uint32_t v;
      while (s >> v) g.graph_inputs.push_back(v);
    } else if (t == "B") {
      CtBundle b;
      unsigned cls = 0, rep = 0;
      s >> b.id >> b.lanes >> b.level >> b.components >> cls >> b.chunk_period >> rep >> b.app_node >> b.tag;
      b.cls = (BundleClass)cls;
      b.replicate_hint = rep != 0;
      if (b.id != g.bundles.size()) throw std::invalid_argument("heops: bundle ids must be dense");
      g.bundles.push_back(b);
    } else if (t == "O") {
      HeOp op;
      unsigned kind = 0, agg = 0;
      int acc = 0, al = 0;
      size_t nin = 0;
      s >> op.id >> kind >> op.rot_offset >> op.out.bundle >> op.out.lane >> op.out.lane_count >> acc >> al >>
          op.phase >> op.work >> op.use_level >> op.app_node >> agg >> nin;
      op.kind = (HeOpKind)kind;
      op.accumulate = acc != 0;
      op.aligned = al != 0;
      op.aggregation = (AggregationAxis)agg;
      for (size_t i = 0; i < nin; ++i) {
        LaneSlice sl;
        s >> sl.bundle >> sl.lane >> sl.lane_count;
        op.ins.push_back(sl);
      }
      if (!s) throw std::invalid_argument("heops: malformed op line");
      g.ops.push_back(op);
    }
  }
  validate_heops(g);
  return g;
}

// Structural checks of a graph from outside the lowering (a heops file or an
// in-memory graph handed over the C-ABI): every index the executor and the
// kernels derive from it must stay inside the bundle table, lane ranges and
// levels.  Violations are std::invalid_argument (AEGIS_EINVAL).
void validate_heops(const HeOpGraph& g) {
  const size_t nb = g.bundles.size();
  auto bad = [](const std::string& m) { throw std::invalid_argument("heops: " + m); };
  for (size_t i = 0; i < nb; ++i) {
    const CtBundle& b = g.bundles[i];
    if (b.id != i) bad("bundle ids must be dense");
    if (b.lanes == 0 || b.components == 0 || b.components > 3) bad("bundle " + std::to_string(i) + " has a bad shape");
    if (b.level == 0 || b.level > 64) bad("bundle " + std::to_string(i) + " level out of range");
  }
  for (uint32_t in : g.graph_inputs)
    if (in >= nb) bad("graph input " + std::to_string(in) + " is not a bundle");
  auto slice_ok = [&](const LaneSlice& s) {
    return s.bundle < nb && s.lane_count > 0 && (uint64_t)s.lane + s.lane_count <= g.bundles[s.bundle].lanes;
  };
  for (const HeOp& op : g.ops) {
    const std::string at = "op " + std::to_string(op.id);
    if ((unsigned)op.kind > (unsigned)HeOpKind::kBoot) bad(at + ": unknown kind");
    if (!slice_ok(op.out)) bad(at + ": output slice outside its bundle");
    if (op.ins.size() > 4) bad(at + ": too many operands");
    if (op.kind != HeOpKind::kEncode && op.use_level == 0) bad(at + ": use_level 0");
    for (const LaneSlice& s : op.ins) {
      if (!slice_ok(s)) bad(at + ": operand slice outside its bundle");
      if (op.use_level > g.bundles[s.bundle].level) bad(at + ": use_level above an operand's level");
    }
    const bool shrinks = op.kind == HeOpKind::kRescale || op.kind == HeOpKind::kBoot || op.kind == HeOpKind::kEncode;
    if (!shrinks && op.use_level > g.bundles[op.out.bundle].level) bad(at + ": use_level above the output's level");
    if (op.kind == HeOpKind::kRescale && op.use_level < 2) bad(at + ": rescale needs two limbs");
    if (op.kind == HeOpKind::kRot && op.rot_offset <= -500) bad(at + ": rotation offset must be > -500 (key id 1000 + r)");
    if (op.kind == HeOpKind::kRescale && g.bundles[op.out.bundle].level + 1 < op.use_level)
      bad(at + ": rescale output level below use_level - 1");
  }
}

}  // namespace aegis::heplan

// shard.cu -- lane ownership propagation (see shard.h).
#include <stdexcept>
#include <string>

#include "shard.h"

namespace aegis {

PcmmShape pcmm_shape(uint32_t in_l, uint32_t out_l, uint32_t w_l, uint32_t chunk) {
  uint64_t tg = 1;
  while (tg * tg * w_l < (uint64_t)in_l * out_l) ++tg;
  if (tg * tg * w_l != (uint64_t)in_l * out_l || in_l % tg || out_l % tg)
    throw std::logic_error("PMult lane shapes inconsistent");
  if (chunk != 0 && chunk < out_l && out_l % chunk != 0)
    throw std::invalid_argument("PMult chunk_period must divide the accumulator lanes");
  PcmmShape s;
  s.tg = (uint32_t)tg;
  s.c_in = in_l / s.tg;
  s.c_out = out_l / s.tg;
  if ((uint64_t)s.c_in * s.c_out != w_l) throw std::logic_error("PMult weight lanes inconsistent");
  s.S = (chunk == 0 || chunk >= out_l) ? 1 : out_l / chunk;
  if (s.c_out % s.S) throw std::logic_error("PMult sub-tensor split inconsistent");
  s.c_sub = s.c_out / s.S;
  s.chunk = chunk;
  return s;
}

bool ShardPlan::owns(uint32_t b, uint32_t lane) const {
  if (!active()) return true;
  const LaneTag t = tags[b][lane];
  if (t.tg < 0) return false;
  if (!owns_tg(t.tg)) return false;
  return m == 1 || part_of(b, t.pos) == part;
}

std::vector<std::pair<uint32_t, uint32_t>> ShardPlan::runs(uint32_t b, uint32_t lane0, uint32_t count) const {
  std::vector<std::pair<uint32_t, uint32_t>> r;
  uint32_t i = lane0;
  const uint32_t end = lane0 + count;
  while (i < end) {
    while (i < end && !owns(b, i)) ++i;
    if (i >= end) break;
    const uint32_t s = i;
    while (i < end && owns(b, i)) ++i;
    r.emplace_back(s, i);
  }
  return r;
}

std::vector<std::pair<uint32_t, uint32_t>> ShardPlan::tg_runs(uint32_t b, uint32_t lane0, uint32_t count) const {
  std::vector<std::pair<uint32_t, uint32_t>> r;
  auto in = [&](uint32_t l) { return !active() || owns_tg(tags[b][l].tg); };
  uint32_t i = lane0;
  const uint32_t end = lane0 + count;
  while (i < end) {
    while (i < end && !in(i)) ++i;
    if (i >= end) break;
    const uint32_t s = i;
    while (i < end && in(i)) ++i;
    r.emplace_back(s, i);
  }
  return r;
}

ShardPlan make_shard_plan(const heplan::HeOpGraph& g, uint32_t tg_total, uint32_t world, uint32_t rank) {
  using K = heplan::HeOpKind;
  if (world == 0 || rank >= world || tg_total == 0) throw std::invalid_argument("bad shard spec");
  ShardPlan P;
  P.tg_total = tg_total;
  P.world = world;
  P.rank = rank;
  if (world <= tg_total) {
    const uint32_t per = (tg_total + world - 1) / world;
    P.tg_lo = std::min(tg_total, rank * per);
    P.tg_hi = std::min(tg_total, P.tg_lo + per);
  } else {
    if (world % tg_total) throw std::invalid_argument("world size must divide or be a multiple of token groups");
    P.m = world / tg_total;
    P.tg_lo = rank / P.m;
    P.tg_hi = P.tg_lo + 1;
    P.part = rank % P.m;
  }
  P.tags.resize(g.bundles.size());
  for (size_t b = 0; b < g.bundles.size(); ++b) P.tags[b].assign(g.bundles[b].lanes, LaneTag{});
  auto set = [&](uint32_t b, uint32_t lane, LaneTag t, const heplan::HeOp& op) {
    LaneTag& cur = P.tags[b][lane];
    if (cur.tg < 0) {
      cur = t;
    } else if (cur.tg != t.tg || cur.pos != t.pos) {
      throw std::logic_error("op " + std::to_string(op.id) + " mixes lanes of different token groups (" +
                             g.bundles[b].tag + ")");
    }
  };
  for (uint32_t in : g.graph_inputs) {
    const uint32_t lanes = g.bundles[in].lanes;
    if (lanes % tg_total) throw std::logic_error("graph input lanes not a multiple of token groups");
    const uint32_t c = lanes / tg_total;
    for (uint32_t l = 0; l < lanes; ++l) P.tags[in][l] = LaneTag{(int32_t)(l / c), (int32_t)(l % c)};
  }
  for (const heplan::HeOp& op : g.ops) {
    if (op.kind == K::kEncode) continue;
    const uint32_t n = op.out.lane_count;
    if (op.kind == K::kPMult) {
      const PcmmShape s = pcmm_shape(op.ins[0].lane_count, n, op.ins[1].lane_count,
                                     g.bundles[op.out.bundle].chunk_period);
      for (uint32_t t = 0; t < s.tg; ++t) {
        for (uint32_t ci = 0; ci < s.c_in; ++ci) {  // inputs must belong to group t
          const LaneTag xt = P.tags[op.ins[0].bundle][op.ins[0].lane + t * s.c_in + ci];
          if (xt.tg != (int32_t)t) throw std::logic_error("PCMM input lane outside its token group");
        }
        for (uint32_t o = 0; o < s.c_out; ++o)
          set(op.out.bundle, op.out.lane + pcmm_lane(s, t, o), LaneTag{(int32_t)t, (int32_t)(o % s.c_sub)}, op);
      }
      continue;
    }
    for (uint32_t l = 0; l < n; ++l) {
      const heplan::LaneSlice& a = op.ins[0];
      const LaneTag src = P.tags[a.bundle][a.lane + (a.lane_count == n ? l : l % a.lane_count)];
      if (src.tg < 0) throw std::logic_error("op " + std::to_string(op.id) + " reads an untagged lane");
      for (size_t k = 1; k < op.ins.size(); ++k) {
        const heplan::LaneSlice& b = op.ins[k];
        const LaneTag o2 = P.tags[b.bundle][b.lane + (b.lane_count == n ? l : l % b.lane_count)];
        if (o2.tg != src.tg) throw std::logic_error("op " + std::to_string(op.id) + " couples token groups");
      }
      set(op.out.bundle, op.out.lane + l, src, op);
    }
  }
  P.npos.assign(g.bundles.size(), 0);
  for (size_t b = 0; b < g.bundles.size(); ++b)
    for (const LaneTag& t : P.tags[b])
      if (t.pos >= 0 && (uint32_t)t.pos + 1 > P.npos[b]) P.npos[b] = (uint32_t)t.pos + 1;
  if (P.m > 1) {
    // A token group split over m ranks is only exact if every lane-local op
    // reads operand lanes owned by the same part as its output lane (PCMM is
    // input-stationary and exempt: its reduce-scatter moves the data).  Shapes
    // whose operands wrap onto fewer positions than the output (e.g. score
    // lanes < output lanes at very small T / N) would read lanes no rank of
    // this part computed: refuse them instead of computing garbage.
    for (const heplan::HeOp& op : g.ops) {
      if (op.kind == K::kEncode || op.kind == K::kPMult) continue;
      const uint32_t n = op.out.lane_count;
      for (uint32_t l = 0; l < n; ++l) {
        const LaneTag ot = P.tags[op.out.bundle][op.out.lane + l];
        const uint32_t want = P.part_of(op.out.bundle, ot.pos);
        for (const heplan::LaneSlice& a : op.ins) {
          const uint32_t il = a.lane + (a.lane_count == n ? l : l % a.lane_count);
          if (P.part_of(a.bundle, P.tags[a.bundle][il].pos) != want)
            throw std::invalid_argument("token group split over " + std::to_string(P.m) + " ranks: op " +
                                        std::to_string(op.id) + " (" + g.bundles[op.out.bundle].tag +
                                        ") reads lanes another rank owns; use world <= token groups (" +
                                        std::to_string(tg_total) + ") for this shape");
        }
      }
    }
  }
  return P;
}

}  // namespace aegis

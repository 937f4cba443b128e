// shard.h -- token-coherent lane ownership for multi-GPU execution.
//
// AEGIS places whole modulus-coherent lanes (every limb of a ciphertext) in
// contiguous token chunks (placement.hpp:175-182, kLaneChunks).  With the
// reference's lane semantics every HE op is lane-local except
// PCMM, which couples lanes only inside one token group.  We therefore tag each
// lane of every bundle with (token group, position) by propagating through the
// op list, and give each rank
//   G <= token groups : whole token groups                -> no data-path collective
//   G  = m * groups   : one token group, positions split in m contiguous parts;
//                       PCMM becomes input-stationary (each rank multiplies its
//                       own input positions into all outputs of the group) and
//                       the partial accumulators are reduce-scattered once per
//                       matmul, just before the rescale ("reduce locally before
//                       send").
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "heplan_ir.h"

namespace aegis {

struct LaneTag {
  int32_t tg = -1, pos = -1;
};

struct ShardPlan {
  uint32_t tg_total = 1, world = 1, rank = 0;
  uint32_t m = 1;  // ranks per token group (world > tg_total)
  uint32_t tg_lo = 0, tg_hi = 1, part = 0;
  std::vector<std::vector<LaneTag>> tags;  // [bundle][lane]
  std::vector<uint32_t> npos;              // [bundle] positions per token group

  bool active() const { return world > 1; }
  uint32_t part_of(uint32_t b, int32_t pos) const { return npos[b] ? (uint32_t)pos * m / npos[b] : 0; }
  bool owns(uint32_t b, uint32_t lane) const;
  bool owns_tg(int32_t tg) const { return tg >= (int32_t)tg_lo && tg < (int32_t)tg_hi; }
  // maximal contiguous runs [start, end) of owned lanes inside [lane0, lane0 + count)
  std::vector<std::pair<uint32_t, uint32_t>> runs(uint32_t b, uint32_t lane0, uint32_t count) const;
  // the same over every lane of this rank's token groups (all m parts): the
  // lanes a gather-mode PCMM computes on every rank of the group
  std::vector<std::pair<uint32_t, uint32_t>> tg_runs(uint32_t b, uint32_t lane0, uint32_t count) const;
};

// Tags every bundle lane; throws std::logic_error if an op mixes token groups
// (which would require a collective this placement does not plan for).
ShardPlan make_shard_plan(const heplan::HeOpGraph& g, uint32_t tg_total, uint32_t world, uint32_t rank);

// PMult lane shapes: token groups, c_in, c_out, sub-tensor count, c_sub
struct PcmmShape {
  uint32_t tg, c_in, c_out, S, c_sub, chunk;
};
PcmmShape pcmm_shape(uint32_t in_lanes, uint32_t out_lanes, uint32_t w_lanes, uint32_t chunk_period);
// accumulator lane of (token group t, output o)
inline uint32_t pcmm_lane(const PcmmShape& s, uint32_t t, uint32_t o) {
  return s.S == 1 ? t * s.c_out + o : (o / s.c_sub) * s.chunk + t * s.c_sub + o % s.c_sub;
}

}  // namespace aegis

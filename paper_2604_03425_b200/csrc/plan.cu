// plan.cu -- Aegis execution-plan compiler (see plan.h).
#include <algorithm>
#include <map>
#include <stdexcept>

#include "plan.h"
#include "shard.h"

namespace aegis {

namespace hp = heplan;
using K = hp::HeOpKind;

CommCategory category_of(const std::string& tag) {  // comm_plan.hpp:36-49 by app-node name
  auto has = [&](const char* s) { return tag.find(s) != std::string::npos; };
  if (has(".boot")) return CommCategory::kBoot;
  if (has(".qkv") || has(".out_proj") || has(".ffn1") || has(".ffn2")) return CommCategory::kFfn;
  if (has(".score") || has(".softmax") || has(".att_out")) return CommCategory::kAttention;
  if (has(".layer_norm")) return CommCategory::kLayerNorm;
  return CommCategory::kOther;
}

int64_t pcmm_activation_op(const hp::HeOpGraph& g, uint32_t acc) {
  std::vector<char> rot_out(g.bundles.size(), 0);
  for (const hp::HeOp& op : g.ops)
    if (op.kind == K::kRot) rot_out[op.out.bundle] = 1;
  for (size_t i = 0; i < g.ops.size(); ++i)
    if (g.ops[i].kind == K::kPMult && g.ops[i].out.bundle == acc && !rot_out[g.ops[i].ins[0].bundle])
      return (int64_t)i;
  return -1;
}

bool gather_executed(const hp::HeOpGraph& g, uint32_t acc, uint32_t first_pmult_op) {
  const hp::HeOp& pm = g.ops[first_pmult_op];
  const PcmmShape sh = pcmm_shape(pm.ins[0].lane_count, pm.out.lane_count, pm.ins[1].lane_count,
                                  g.bundles[acc].chunk_period);
  return (uint64_t)sh.c_in * g.bundles[pm.ins[0].bundle].level <= (uint64_t)sh.c_out * g.bundles[acc].level;
}

ExecPlan build_plan(const hp::HeOpGraph& g, uint32_t tg_total, uint32_t world, uint32_t ring_degree, bool reorder,
                    bool reference_modes) {
  if (world == 0 || tg_total == 0) throw std::invalid_argument("plan: world and token groups must be positive");
  ExecPlan P;
  P.world = world;
  P.tg_total = tg_total;
  P.m = world > tg_total ? world / tg_total : 1;
  P.reordered = reorder;
  const uint64_t limb = (uint64_t)ring_degree * 8;
  std::vector<ShardPlan> sp;
  try {
    for (uint32_t r = 0; r < world; ++r) sp.push_back(world > 1 ? make_shard_plan(g, tg_total, world, r) : ShardPlan{});
  } catch (const std::exception& e) {
    P.executable = false;
    P.note = e.what();
    sp.clear();
  }

  // producers, last PMult per accumulator, the matmuls
  std::vector<int64_t> producer(g.bundles.size(), -1), last_pmult(g.bundles.size(), -1),
      first_pmult(g.bundles.size(), -1);
  for (size_t i = 0; i < g.ops.size(); ++i) {
    const hp::HeOp& op = g.ops[i];
    if (producer[op.out.bundle] < 0) producer[op.out.bundle] = (int64_t)i;
    if (op.kind == K::kPMult) {
      last_pmult[op.out.bundle] = (int64_t)i;
      if (first_pmult[op.out.bundle] < 0) first_pmult[op.out.bundle] = (int64_t)i;
    }
  }

  // gather-mode matmuls (reference_modes): the activation and its rotations are
  // computed on every lane of the token group, each device its own output share
  std::vector<char> gather(g.bundles.size(), 0), full_tg(g.bundles.size(), 0), cmult_out(g.bundles.size(), 0);
  for (const hp::HeOp& op : g.ops)
    if (op.kind == K::kCMult) cmult_out[op.out.bundle] = 1;
  if (reference_modes && P.m > 1 && P.executable)
    for (size_t b = 0; b < g.bundles.size(); ++b) {
      const int64_t act = first_pmult[b] < 0 ? -1 : pcmm_activation_op(g, (uint32_t)b);
      if (act < 0 || !gather_executed(g, (uint32_t)b, (uint32_t)act)) continue;
      gather[b] = 1;
      const hp::HeOp& pm0 = g.ops[act];
      const uint32_t x = pm0.ins[0].bundle;
      full_tg[x] = 1;  // (when x is a boot output the boot runs on every lane of the group)
      for (const hp::HeOp& op : g.ops)
        if (op.kind == K::kRot && op.ins[0].bundle == x && op.app_node == pm0.app_node) full_tg[op.out.bundle] = 1;
    }
  auto comps_alloc = [&](uint32_t b) { return cmult_out[b] ? 3u : std::max(2u, g.bundles[b].components); };

  // ---- compute streams ------------------------------------------------------
  P.devices.resize(P.executable ? world : 0);
  std::vector<std::map<int64_t, uint32_t>> first_pos(world), last_pos(world);  // op -> compute position
  for (uint32_t d = 0; d < (uint32_t)P.devices.size(); ++d) {
    DevicePlan& D = P.devices[d];
    for (size_t i = 0; i < g.ops.size(); ++i) {
      const hp::HeOp& op = g.ops[i];
      std::vector<std::pair<uint32_t, uint32_t>> runs;
      uint8_t flags = 0;
      if (world == 1 || op.kind == K::kEncode) {
        runs.emplace_back(op.out.lane, op.out.lane + op.out.lane_count);
      } else if (op.kind == K::kPMult && P.m > 1 && gather[op.out.bundle]) {
        // every input of the group, this device's share of every sub-tensor's outputs
        const PcmmShape sh = pcmm_shape(op.ins[0].lane_count, op.out.lane_count, op.ins[1].lane_count,
                                        g.bundles[op.out.bundle].chunk_period);
        const uint32_t share = sh.c_sub / P.m;
        for (uint32_t s = 0; s < sh.S; ++s) {
          const uint32_t l0 = op.out.lane + pcmm_lane(sh, sp[d].tg_lo, s * sh.c_sub + sp[d].part * share);
          runs.emplace_back(l0, l0 + share);
        }
      } else if (full_tg[op.out.bundle]) {
        runs = sp[d].tg_runs(op.out.bundle, op.out.lane, op.out.lane_count);
      } else if (op.kind == K::kPMult && P.m > 1) {
        // input-stationary partial sums into every output lane of the group
        const PcmmShape sh = pcmm_shape(op.ins[0].lane_count, op.out.lane_count, op.ins[1].lane_count,
                                        g.bundles[op.out.bundle].chunk_period);
        for (uint32_t s = 0; s < sh.S; ++s) {
          const uint32_t l0 = op.out.lane + pcmm_lane(sh, sp[d].tg_lo, s * sh.c_sub);
          runs.emplace_back(l0, l0 + sh.c_sub);
        }
        flags = 2;
      } else {
        runs = sp[d].runs(op.out.bundle, op.out.lane, op.out.lane_count);
      }
      for (auto [a, e] : runs) {
        if (!first_pos[d].count((int64_t)i)) first_pos[d][(int64_t)i] = (uint32_t)D.compute.size();
        last_pos[d][(int64_t)i] = (uint32_t)D.compute.size();
        D.compute.push_back(PlanInstr{(uint32_t)i, a, e - a, flags, -1});
      }
    }
  }

  // ---- matmuls: mode analysis + the executed reduce-scatter events ----------
  for (size_t b = 0; b < g.bundles.size(); ++b) {
    if (first_pmult[b] < 0) continue;
    const int64_t act = pcmm_activation_op(g, (uint32_t)b);
    const hp::HeOp& pm0 = g.ops[act >= 0 ? act : first_pmult[b]];
    const hp::HeOp& pml = g.ops[last_pmult[b]];
    MatmulInfo mi;
    mi.app_node = pm0.app_node;
    mi.acc_bundle = (uint32_t)b;
    mi.input_bundle = pm0.ins[0].bundle;
    mi.ship_bundle = mi.input_bundle;
    mi.tag = g.bundles[b].tag;
    uint32_t ship_level = g.bundles[mi.input_bundle].level;
    const int64_t pr = producer[mi.input_bundle];
    if (pr >= 0 && g.ops[pr].kind == K::kBoot) {  // send before bootstrapping
      mi.ship_bundle = g.ops[pr].ins[0].bundle;
      ship_level = g.ops[pr].use_level;
    }
    const PcmmShape sh = pcmm_shape(pml.ins[0].lane_count, pml.out.lane_count, pml.ins[1].lane_count,
                                    g.bundles[b].chunk_period);
    const uint32_t level = g.bundles[b].level, m = P.m;
    if (m > 1) {
      // NCCL-style volumes: every device receives (m-1)/m of the group's buffer
      mi.gather_bytes = (uint64_t)tg_total * (m - 1) * sh.c_in * ship_level * 2 * limb;
      mi.reduce_bytes = (uint64_t)tg_total * (m - 1) * sh.c_out * level * 2 * limb;
      mi.chosen = mi.gather_bytes <= mi.reduce_bytes ? MatmulMode::kGatherInputs : MatmulMode::kReduceOutputs;
      mi.executed = !P.executable ? MatmulMode::kLocal
                    : gather[b]       ? MatmulMode::kGatherInputs
                                      : MatmulMode::kReduceOutputs;
      // the rescale (first reader after the last PMult) waits for the exchange
      int64_t reader = -1;
      for (size_t i = (size_t)last_pmult[b] + 1; i < g.ops.size() && reader < 0; ++i)
        for (const hp::LaneSlice& s : g.ops[i].ins)
          if (s.bundle == b) reader = (int64_t)i;
      if (gather[b]) {  // one AllGather of the activation per token group
        uint32_t x = pm0.ins[0].bundle, lane0 = pm0.ins[0].lane;
        int64_t reader_op = (int64_t)g.ops.size();  // the matmul's first op reading x (any order)
        for (size_t i = 0; i < g.ops.size(); ++i)
          if (g.ops[i].app_node == pm0.app_node)
            for (const hp::LaneSlice& sl : g.ops[i].ins)
              if (sl.bundle == x) reader_op = std::min(reader_op, (int64_t)i);
        int64_t producer_op = -1;  // last writer of x before the matmul
        for (int64_t i = 0; i < reader_op; ++i)
          if (g.ops[i].out.bundle == x && g.ops[i].kind != K::kEncode) producer_op = i;
        // send before bootstrapping: the boot's input is shipped, the boot runs on every lane
        if (producer_op >= 0 && g.ops[producer_op].kind == K::kBoot &&
            g.ops[producer_op].ins[0].lane_count == g.ops[producer_op].out.lane_count &&
            g.ops[producer_op].out.lane <= lane0) {
          const hp::HeOp& bo = g.ops[producer_op];
          reader_op = producer_op;
          lane0 = bo.ins[0].lane + (lane0 - bo.out.lane);
          x = bo.ins[0].bundle;
          producer_op = -1;
          for (int64_t i = 0; i < reader_op; ++i)
            if (g.ops[i].out.bundle == x && g.ops[i].kind != K::kEncode) producer_op = i;
        }
        for (uint32_t t = 0; t < tg_total; ++t) {
          PlanEvent e;
          e.id = (uint32_t)P.events.size();
          e.kind = CollKind::kAllGather;
          e.semantic = CollSemantic::kMove;
          e.dev_lo = t * m;
          e.dev_count = m;
          e.bundle = x;
          e.lane = lane0 + t * sh.c_in;
          e.lane_count = sh.c_in;
          e.level = g.bundles[x].level;
          e.comps = comps_alloc(x);
          e.bytes_per_device = (uint64_t)(m - 1) * (sh.c_in / m) * e.level * e.comps * limb;
          e.bytes_total = e.bytes_per_device * m;
          e.app_node = pm0.app_node;
          e.he_op = producer_op >= 0 ? (uint32_t)producer_op : 0;
          e.category = category_of(g.bundles[b].tag);
          e.executed = true;
          for (uint32_t dd = e.dev_lo; dd < e.dev_lo + m; ++dd) {
            e.trigger_pos.push_back(producer_op >= 0 && last_pos[dd].count(producer_op) ? last_pos[dd].at(producer_op)
                                                                                        : 0);
            const uint32_t w = first_pos[dd].count(reader_op) ? first_pos[dd].at(reader_op) : UINT32_MAX;
            e.wait_pos.push_back(w);
            if (w != UINT32_MAX && P.devices[dd].compute[w].wait_event < 0)
              P.devices[dd].compute[w].wait_event = (int32_t)e.id;
            P.devices[dd].comm.push_back(e.id);
          }
          P.events.push_back(e);
        }
        P.matmuls.push_back(mi);
        continue;
      }
      for (uint32_t t = 0; t < (P.executable ? tg_total : 0); ++t)
        for (uint32_t s = 0; s < sh.S; ++s) {
          PlanEvent e;
          e.id = (uint32_t)P.events.size();
          e.kind = CollKind::kReduceScatter;
          e.semantic = CollSemantic::kCombineScatter;
          e.dev_lo = t * m;
          e.dev_count = m;
          e.bundle = (uint32_t)b;
          e.lane = pml.out.lane + pcmm_lane(sh, t, s * sh.c_sub);
          e.lane_count = sh.c_sub;
          e.level = level;
          e.bytes_per_device = (uint64_t)(m - 1) * (sh.c_sub / m) * level * 2 * limb;
          e.bytes_total = e.bytes_per_device * m;
          e.app_node = pml.app_node;
          e.he_op = (uint32_t)last_pmult[b];
          e.category = category_of(g.bundles[b].tag);
          e.executed = true;
          for (uint32_t d = e.dev_lo; d < e.dev_lo + m; ++d) {
            e.trigger_pos.push_back(last_pos[d].at(last_pmult[b]));
            // the reader's instruction over this device's share of the sub-tensor waits
            const uint32_t share = sh.c_sub / m, mine = e.lane + (d - e.dev_lo) * share;
            uint32_t w = UINT32_MAX;
            if (reader >= 0 && first_pos[d].count(reader)) {
              const hp::HeOp& rop = g.ops[reader];
              for (uint32_t pos = first_pos[d].at(reader); pos <= last_pos[d].at(reader); ++pos) {
                const PlanInstr& in = P.devices[d].compute[pos];
                // reader lanes map to accumulator lanes one-for-one (rescale of the accumulator)
                const uint32_t a0 = rop.ins.empty() ? in.lane : rop.ins[0].lane + (in.lane - rop.out.lane);
                if (a0 < mine + share && mine < a0 + in.lane_count) {
                  w = pos;
                  break;
                }
              }
            }
            e.wait_pos.push_back(w);
            if (w != UINT32_MAX && P.devices[d].compute[w].wait_event < 0) P.devices[d].compute[w].wait_event = (int32_t)e.id;
            P.devices[d].comm.push_back(e.id);
          }
          P.events.push_back(e);
        }
    } else {
      mi.chosen = mi.executed = MatmulMode::kLocal;
    }
    P.matmuls.push_back(mi);
  }

  // ---- staggered diagonal order: part p starts at offset p * 64 / m
  if (reorder && P.m > 1 && P.executable) {
    for (uint32_t d = 0; d < world; ++d) {
      const uint32_t part = d % P.m;
      std::vector<PlanInstr>& C = P.devices[d].compute;
      for (const MatmulInfo& mi : P.matmuls) {
        // the matmul's diagonal ops: phase >= 0 ops of its app node between the first PMult's
        // rotation source and the last PMult
        size_t lo = C.size(), hi = 0;
        int maxph = 0;
        for (size_t k = 0; k < C.size(); ++k) {
          const hp::HeOp& op = g.ops[C[k].op];
          if (op.app_node != mi.app_node || op.phase < 0 || op.kind == K::kRescale) continue;
          if (op.kind != K::kRot && op.kind != K::kPMult && op.kind != K::kEncode) continue;
          lo = std::min(lo, k);
          hi = std::max(hi, k + 1);
          maxph = std::max(maxph, op.phase);
        }
        if (lo >= hi) continue;
        const int period = maxph + 1, shift = (int)(part * (uint32_t)period / P.m);
        std::stable_sort(C.begin() + (long)lo, C.begin() + (long)hi, [&](const PlanInstr& a, const PlanInstr& b) {
          const int pa = g.ops[a.op].phase < 0 ? 0 : g.ops[a.op].phase, pb = g.ops[b.op].phase < 0 ? 0 : g.ops[b.op].phase;
          return (pa - shift + period) % period < (pb - shift + period) % period;
        });
      }
    }
    // positions moved: recompute event triggers / waits
    for (PlanEvent& e : P.events)
      for (uint32_t k = 0; k < e.dev_count; ++k) {
        const DevicePlan& D = P.devices[e.dev_lo + k];
        uint32_t trig = 0;
        for (uint32_t pos = 0; pos < D.compute.size(); ++pos)
          if (D.compute[pos].op == e.he_op || (g.ops[D.compute[pos].op].kind == K::kPMult &&
                                               g.ops[D.compute[pos].op].out.bundle == e.bundle))
            trig = std::max(trig, pos);
        e.trigger_pos[k] = trig;
        for (uint32_t pos = 0; pos < D.compute.size(); ++pos)
          if (D.compute[pos].wait_event == (int32_t)e.id) e.wait_pos[k] = pos;
      }
  }
  return P;
}

}  // namespace aegis

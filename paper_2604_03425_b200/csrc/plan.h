// plan.h -- the Aegis execution plan (comm_plan.hpp:51-118 ExecutionPlan /
// DevicePlan / PlanInstr / CollectiveEvent, rebuilt for this executor).
//
// build_plan walks the HE-op graph under token-coherent placement (shard.h)
// and emits, per device, the compute instructions (HeOp, owned lane runs) and
// the collective events with their trigger (compute position that must retire
// first) and wait (compute position that may not start before the event) --
// the two-stream contract of PAPER.md:514-527 that the executor realises with
// the comm stream and CUDA events (executor.cu reduce_async).
//
// Collective insertion follows PAPER.md:481-497 and comm_plan.hpp:194-242:
//   * only PCMM couples lanes, and only inside a token group,
//     so events exist only when a token group spans m > 1 devices;
//   * per matmul the cheaper of kGatherInputs (AllGather of the activation,
//     "send before bootstrapping": the pre-boot bundle when the activation is
//     a boot output) and kReduceOutputs (ReduceScatter of the partial
//     accumulators, "reduce locally before send") is chosen by bytes, exactly
//     the reference's rule (comm_plan.hpp:226-238);
//   * "rescale before send" cannot apply to partial sums (the rescale rounds;
//     rounding does not commute with the sum), so reductions precede rescale.
// The executor implements kReduceOutputs (input-stationary PCMM, no duplicated
// rotations); `executed` marks the events it runs, and the plan records the
// bytes of both modes per matmul so the reference's choice can be compared.
// `reorder` staggers the diagonal (rotation-offset) order per device part,
// as PAPER.md:525 describes; with bundled PMults every diagonal feeds every
// output, so the stagger changes no event trigger of the reduce mode (it is
// recorded in the plan for the gather mode, where it does).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "heplan_ir.h"

namespace aegis {

enum class CollKind : uint8_t { kAllGather, kReduceScatter, kAllReduce };
enum class CollSemantic : uint8_t { kMove, kCombine, kCombineScatter };  // comm_plan.hpp:52-56
enum class CommCategory : uint8_t { kFfn, kAttention, kLayerNorm, kBoot, kOther };  // comm_plan.hpp:30-49
enum class MatmulMode : uint8_t { kLocal, kGatherInputs, kReduceOutputs };

struct PlanEvent {
  uint32_t id = 0;
  CollKind kind = CollKind::kReduceScatter;
  CollSemantic semantic = CollSemantic::kCombineScatter;
  uint32_t dev_lo = 0, dev_count = 0;  // participants [dev_lo, dev_lo + dev_count)
  uint32_t bundle = 0, lane = 0, lane_count = 0, level = 0, comps = 2;
  uint64_t bytes_per_device = 0, bytes_total = 0;
  uint32_t app_node = 0, he_op = 0;  // the op whose retirement triggers it
  CommCategory category = CommCategory::kOther;
  bool executed = false;  // the executor's data plane runs this event
  std::vector<uint32_t> trigger_pos;  // per participant: compute position that retires first
  std::vector<uint32_t> wait_pos;     // per participant: compute position that waits for it
};

struct PlanInstr {
  uint32_t op = 0;             // HeOp index
  uint32_t lane = 0, lane_count = 0;  // owned output lanes (one run)
  uint8_t flags = 0;           // 2 = accumulates into a partial (per-device) copy
  int32_t wait_event = -1;
};

struct DevicePlan {
  std::vector<PlanInstr> compute;
  std::vector<uint32_t> comm;  // event ids in issue order
};

struct MatmulInfo {
  uint32_t app_node = 0, acc_bundle = 0, input_bundle = 0, ship_bundle = 0;
  MatmulMode chosen = MatmulMode::kLocal;   // the reference's byte rule
  MatmulMode executed = MatmulMode::kLocal; // what this executor runs
  uint64_t gather_bytes = 0, reduce_bytes = 0;  // total over devices, per mode
  std::string tag;
};

struct ExecPlan {
  uint32_t world = 1, tg_total = 1, m = 1;
  bool reordered = false;
  // false when token-coherent placement cannot split this shape over `world`
  // devices (make_shard_plan refuses it); the matmul analysis is still filled
  bool executable = true;
  std::string note;
  std::vector<DevicePlan> devices;
  std::vector<PlanEvent> events;
  std::vector<MatmulInfo> matmuls;
};

// reference_modes: run each matmul in the mode the reference's byte rule picks
// (gather the activation when that moves fewer bytes than reducing the
// outputs; the activation itself is shipped, not a pre-boot form) -- the
// executor's aegis_graph_set_matmul_modes(g, 1); otherwise always reduce
ExecPlan build_plan(const heplan::HeOpGraph& g, uint32_t tg_total, uint32_t world, uint32_t ring_degree,
                    bool reorder, bool reference_modes = false);
// the executed choice for the accumulator `acc` when reference_modes is on:
// gather iff c_in * level(activation) <= c_out * level(acc)
bool gather_executed(const heplan::HeOpGraph& g, uint32_t acc, uint32_t first_pmult_op);
// the PMult of accumulator `acc` that reads the activation itself (its r = 0
// diagonal: the input is not a rotation output) -- independent of op order,
// so staggered graphs (aegis_graph_from_plan) resolve the same activation; -1 if none
int64_t pcmm_activation_op(const heplan::HeOpGraph& g, uint32_t acc);
CommCategory category_of(const std::string& bundle_tag);

}  // namespace aegis

// executor.h -- runs a bundled HE-op graph (he_ir.hpp:57-120) on one GPU:
// SPEC.md:407-415 exec_sequential, plus exec_plan-style lane sharding for
// multi-GPU token-coherent placement (shard.h).
#pragma once

#include <vector>

#include "context.h"
#include "heplan_ir.h"
#include "p2p.h"
#include "shard.h"

namespace aegis {

// Reduce-scatter hook for sharded PCMM (world > token groups): sum the
// `words_per_rank * m` words at `buf` across the m ranks of token group `group`
// and leave this rank's share (ncclUint64 sum semantics) at `buf + part * words_per_rank`.
// Called with the compute stream idle; must return after the data is in place.
typedef int (*ReduceFn)(void* user, u64* buf, uint64_t words_per_rank, uint32_t group);

struct RunOptions {
  int64_t max_ops = -1;
  unsigned long long* d_hash = nullptr;  // per-bundle hash slots (owned lanes only)
  const u64* host_in = nullptr;          // graph inputs from host memory
  u64* host_out = nullptr;               // final bundle to host memory
  const ShardPlan* shard = nullptr;
  // if set, bundle hashes cover only the lanes this plan owns (execution is
  // unaffected): the unsharded run reports one token group's lanes
  const ShardPlan* hash_lanes = nullptr;
  ReduceFn reduce = nullptr;
  void* reduce_user = nullptr;
  // device-synchronised reduce-scatter window (p2p.h): when set, sharded PCMM
  // sums are exchanged on the comm stream as soon as the last PMult of the
  // accumulator is issued, one exchange per sub-tensor, with CUDA-event edges
  // back to the compute stream (no host callback, no host barrier)
  P2pWindow* p2p = nullptr;
  int fault = 0;  // fault injection (tests): 1 = drop the PCMM exchange (each rank keeps its partial sums)
  // stored-plaintext PCMM (SURVEY §8(d) variant, §8(f) rank 4): every Encode op
  // writes its weight bundle to HBM (kGenerate rows, 1 component) and the PMult
  // kernel reads it instead of generating the weights in registers; every
  // ciphertext bundle is bit-identical to the fused form (weight bundles are
  // not hashed, as in the oracle, which never materialises them)
  bool stored_weights = false;
  // reference_modes (needs `p2p`): a matmul whose activation is cheaper to
  // gather than its partial outputs are to reduce (plan.h gather_executed) runs
  // output-stationary: the activation is all-gathered over the token group on
  // the comm stream, every rank rotates all of its lanes and computes its own
  // output share completely -- no reduction (comm_plan.hpp:226-238 kGatherInputs)
  bool reference_modes = false;
  bool hoist = true;
  bool dce = false;  // skip output lanes no later op reads (final bundle unchanged)
  bool wrap_defer = true;  // wrapped accumulating CAdds summed at the operand's width (bit-identical)
  std::vector<float>* op_ms = nullptr;  // if set: per-op device time (CUDA events)
  // if set (with op_ms): every comm-stream exchange as (start ms, end ms, bundle)
  // relative to the run's first compute-stream event -- the two-stream trace
  std::vector<float>* comm_trace = nullptr;
};

class Executor {
 public:
  Executor(Context& c, const heplan::HeOpGraph& g, const RunOptions& opt);
  ~Executor();
  void run();
  size_t h2d_bytes = 0, d2h_bytes = 0, comm_bytes = 0;

 private:
  struct Group {  // Rot ops sharing one source (hoisted ModUp)
    u32 src, lane0, count, level;
    int64_t last = -1;
    u32 size = 0;
    u64* ext = nullptr;
    bool prepared = false;
    std::vector<std::pair<u32, u32>> runs;  // owned source runs (absolute lanes)
    std::vector<u32> run_off;               // compact ext offset (lanes) of each run
    u32 hoisted = 0;                        // lanes (in run order) whose ModUp is cached
    std::vector<char> src_live;             // dce: source lanes some rotation of the group needs
  };

  Bundle& get(u32 id);
  Bundle& input(const heplan::LaneSlice& s, u32 lo = 0, u32 hi = ~0u);
  void retire(u32 id);
  void hash_bundle(u32 id, const Bundle& b);
  void find_hoist_groups();
  void find_live_lanes();
  bool live_lane(u32 b, u32 lane) const { return !o.dce || live[b][lane]; }
  size_t hoist_budget(size_t out_bytes);
  void step(const heplan::HeOp& op, int64_t i);
  void pmult(const heplan::HeOp& op, int64_t i);
  void reduce_async(u32 bundle);
  void allgather(u32 bundle);  // gather-mode activation: all lanes of the token group
  // compute stream waits for the comm-stream exchanges of `bundle` that cover
  // lanes [lo, hi) (all of them by default)
  void wait_pending(u32 bundle, u32 lo = 0, u32 hi = ~0u);
  void rot_run(const heplan::HeOp& op, int64_t i, u32 r0, u32 len);
  void reduce_partial(u32 bundle);
  void donate(const heplan::HeOp& op, int64_t i);
  bool wrap_deferrable(const heplan::HeOp& op) const;
  void materialize(u32 bundle);
  std::vector<std::pair<u32, u32>> out_runs(const heplan::HeOp& op) const;
  static LaneMap sub_map(const heplan::LaneSlice& s, u32 n, u32 pos, u32 len);
  u32 wrap_end(const heplan::HeOp& op, u32 pos, u32 end) const;

  Context& c;
  const heplan::HeOpGraph& g;
  RunOptions o;
  std::vector<Bundle*> buf;
  std::vector<u32> alloc_comps, cur_comps;
  std::vector<char> zero_first, partial, donated, is_weight;
  std::vector<char> gather_acc, full_tg, gather_src;  // reference_modes bookkeeping (see RunOptions)
  std::vector<u32> gather_lane0, gather_cin;          // gathered bundle: lane of (tg 0, pos 0), lanes per tg
  std::vector<int64_t> first_pmult;
  std::vector<int64_t> last_use, last_pmult;
  struct Pending {
    u32 lo, hi;
    cudaEvent_t ev;
  };
  std::vector<std::vector<Pending>> pending;  // comm-stream exchanges not yet waited for
  std::vector<cudaEvent_t> events;            // every event this run created (destroyed at the end)
  struct CommMark {
    cudaEvent_t start, end;
    u32 bundle;
  };
  std::vector<CommMark> comm_marks;  // comm_trace: timed exchanges
  void comm_mark_begin(u32 bundle);
  void comm_mark_end();
  std::vector<Group> groups;
  std::vector<int> group_of;
  std::vector<std::vector<char>> live;  // dce: [bundle][lane] read by a later op (or final)
  std::vector<Bundle*> shadow;          // wrap_defer: pending sum S of a bundle's wrapped addends
  std::vector<u32> shadow_level;
  u32 final_bundle = 0xffffffffu;
};

}  // namespace aegis

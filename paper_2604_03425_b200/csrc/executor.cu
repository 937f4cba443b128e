// executor.cu -- HE-op graph executor (see executor.h).
//
// Replays the reference's op list verbatim (he_ir.hpp:683 output), op by op
// on the context stream.  Memory: a bundle is allocated when first written
// (zeroed only if its first writer accumulates) and freed after its last use.
// Rotations reading the same source between writes form a group whose ModUp is
// computed once (bit-exact hoisting).  Under a ShardPlan every
// op touches only the lanes this rank owns; PCMM with several ranks per token
// group accumulates partial sums that are reduce-scattered before the rescale.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <set>

#include "executor.h"
#include "plan.h"

namespace aegis {

namespace hp = heplan;

Executor::Executor(Context& ctx, const hp::HeOpGraph& graph, const RunOptions& opt)
    : c(ctx), g(graph), o(opt) {
  const size_t nb = g.bundles.size();
  buf.assign(nb, nullptr);
  alloc_comps.resize(nb);
  cur_comps.assign(nb, 0);
  zero_first.assign(nb, 0);
  partial.assign(nb, 0);
  donated.assign(nb, 0);
  is_weight.assign(nb, 0);
  shadow.assign(nb, nullptr);
  shadow_level.assign(nb, 0);
  last_use.assign(nb, -1);
  last_pmult.assign(nb, -1);
  pending.assign(nb, {});
  std::vector<char> seen(nb, 0);
  for (size_t i = 0; i < nb; ++i) alloc_comps[i] = g.bundles[i].components;
  for (size_t i = 0; i < g.ops.size(); ++i) {
    const hp::HeOp& op = g.ops[i];
    last_use[op.out.bundle] = (int64_t)i;
    for (auto& s : op.ins) last_use[s.bundle] = (int64_t)i;
    if (op.kind == hp::HeOpKind::kCMult) alloc_comps[op.out.bundle] = 3;
    if (op.kind == hp::HeOpKind::kPMult) last_pmult[op.out.bundle] = (int64_t)i;
    if (op.kind == hp::HeOpKind::kEncode) is_weight[op.out.bundle] = 1;
    if (!seen[op.out.bundle] && op.kind != hp::HeOpKind::kEncode) {
      seen[op.out.bundle] = 1;
      zero_first[op.out.bundle] = op.accumulate ? 1 : 0;
    }
  }
  if (o.shard && !o.shard->active()) o.shard = nullptr;
  gather_acc.assign(nb, 0);
  full_tg.assign(nb, 0);
  gather_src.assign(nb, 0);
  gather_lane0.assign(nb, 0);
  gather_cin.assign(nb, 0);
  first_pmult.assign(nb, -1);
  for (size_t i = 0; i < g.ops.size(); ++i)
    if (g.ops[i].kind == hp::HeOpKind::kPMult && first_pmult[g.ops[i].out.bundle] < 0)
      first_pmult[g.ops[i].out.bundle] = (int64_t)i;
  if (o.reference_modes && o.shard && o.shard->m > 1) {
    if (!o.p2p) throw Error(AEGIS_EINVAL, "matmul reference modes need a p2p window (aegis_graph_set_p2p)");
    for (size_t b = 0; b < nb; ++b) {
      const int64_t act = first_pmult[b] < 0 ? -1 : pcmm_activation_op(g, (u32)b);
      if (act < 0 || !gather_executed(g, (u32)b, (u32)act)) continue;
      gather_acc[b] = 1;
      const hp::HeOp& pm0 = g.ops[act];
      const u32 x = pm0.ins[0].bundle;
      const PcmmShape sh = pcmm_shape(pm0.ins[0].lane_count, pm0.out.lane_count, pm0.ins[1].lane_count,
                                      g.bundles[b].chunk_period);
      full_tg[x] = 1;
      for (const hp::HeOp& op : g.ops)
        if (op.kind == hp::HeOpKind::kRot && op.ins[0].bundle == x && op.app_node == pm0.app_node)
          full_tg[op.out.bundle] = 1;
      // "send before bootstrapping": when the activation is a
      // boot output, gather the boot's input (fewer limbs) and run the boot on
      // every lane of the group instead
      int64_t prod = -1, first_read = (int64_t)g.ops.size();  // producer: the last writer before the matmul reads x
      for (size_t i = 0; i < g.ops.size(); ++i)
        if (g.ops[i].app_node == pm0.app_node)
          for (const hp::LaneSlice& sl : g.ops[i].ins)
            if (sl.bundle == x) first_read = std::min(first_read, (int64_t)i);
      for (int64_t i = 0; i < first_read; ++i)
        if (g.ops[i].out.bundle == x) prod = i;
      const bool via_boot = prod >= 0 && g.ops[prod].kind == hp::HeOpKind::kBoot &&
                            g.ops[prod].ins[0].lane_count == g.ops[prod].out.lane_count &&
                            g.ops[prod].out.lane <= pm0.ins[0].lane;
      const u32 src = via_boot ? g.ops[prod].ins[0].bundle : x;
      gather_src[src] = 1;
      gather_lane0[src] = via_boot ? g.ops[prod].ins[0].lane + (pm0.ins[0].lane - g.ops[prod].out.lane) : pm0.ins[0].lane;
      gather_cin[src] = sh.c_in;
    }
  }
  if (o.hash_lanes && o.shard) throw Error(AEGIS_EINVAL, "hash lane selection applies to unsharded runs only");
  find_hoist_groups();
  if (o.dce) find_live_lanes();
}

// Backward pass: a lane is live if the final bundle contains it or a later op
// reads it (emit_per_lane operand rule, he_ir.hpp:200-222; a PMult reads every
// input lane of its token groups, taken conservatively as all input lanes).
// Overwrites are not tracked, so the set is a superset of the truly needed lanes.
void Executor::find_live_lanes() {
  using K = hp::HeOpKind;
  live.assign(g.bundles.size(), {});
  for (size_t b = 0; b < g.bundles.size(); ++b) live[b].assign(g.bundles[b].lanes, 0);
  if (g.ops.empty()) return;
  std::fill(live[g.ops.back().out.bundle].begin(), live[g.ops.back().out.bundle].end(), 1);
  for (int64_t i = (int64_t)g.ops.size() - 1; i >= 0; --i) {
    const hp::HeOp& op = g.ops[i];
    if (op.kind == K::kEncode) continue;
    const u32 n = op.out.lane_count;
    const std::vector<char>& lo = live[op.out.bundle];
    bool any = false;
    for (u32 l = 0; l < n; ++l) any = any || lo[op.out.lane + l];
    if (!any) continue;
    for (const hp::LaneSlice& s : op.ins) {
      if (g.bundles[s.bundle].components == 1 && op.kind == K::kPMult) continue;  // kGenerate weights
      std::vector<char>& li = live[s.bundle];
      if (op.kind == K::kPMult) {
        for (u32 k = 0; k < s.lane_count; ++k) li[s.lane + k] = 1;
        continue;
      }
      for (u32 l = 0; l < n; ++l)
        if (lo[op.out.lane + l]) li[s.lane + (s.lane_count == n ? l : l % s.lane_count)] = 1;
    }
  }
  // hoist groups: the source lanes any rotation of the group needs
  for (size_t i = 0; i < g.ops.size(); ++i) {
    if (group_of[i] < 0) continue;
    const hp::HeOp& op = g.ops[i];
    Group& gr = groups[group_of[i]];
    if (gr.src_live.empty()) gr.src_live.assign(gr.count, 0);
    for (u32 l = 0; l < op.out.lane_count && l < gr.count; ++l)
      if (live[op.out.bundle][op.out.lane + l]) gr.src_live[l] = 1;
  }
}

Executor::~Executor() {
  if (!events.empty()) {  // the comm stream may still read bundles freed below
    cudaStreamSynchronize(c.comm);
    cudaStreamSynchronize(c.stream);
    for (cudaEvent_t e : events) cudaEventDestroy(e);
  }
  for (auto& gr : groups)
    if (gr.ext) c.release(gr.ext);
  for (Bundle* S : shadow) c.free_bundle(S);
  for (size_t i = 0; i < buf.size(); ++i)
    if (buf[i] && !donated[i]) c.free_bundle(buf[i]);
}

Bundle& Executor::get(u32 id) {
  if (!pending[id].empty()) wait_pending(id);
  if (!buf[id]) {
    const hp::CtBundle& cb = g.bundles[id];
    const u32 comps = is_weight[id] ? 1 : std::max<u32>(2, alloc_comps[id]);
    buf[id] = c.new_bundle(cb.lanes, comps, cb.level, zero_first[id] != 0);
    cur_comps[id] = 2;
  }
  return *buf[id];
}

Bundle& Executor::input(const hp::LaneSlice& s, u32 lo, u32 hi) {
  if (shadow[s.bundle]) materialize(s.bundle);
  if (!buf[s.bundle]) throw Error(AEGIS_ELOGIC, "op reads bundle " + g.bundles[s.bundle].tag + " before it is written");
  if (partial[s.bundle]) reduce_partial(s.bundle);
  if (!pending[s.bundle].empty()) wait_pending(s.bundle, lo, hi);
  return *buf[s.bundle];
}

void Executor::comm_mark_begin(u32 b) {
  if (!o.comm_trace) return;
  CommMark m{nullptr, nullptr, b};
  AEGIS_CHECK_CUDA(cudaEventCreate(&m.start));
  AEGIS_CHECK_CUDA(cudaEventCreate(&m.end));
  AEGIS_CHECK_CUDA(cudaEventRecord(m.start, c.comm));
  comm_marks.push_back(m);
}
void Executor::comm_mark_end() {
  if (!o.comm_trace || comm_marks.empty()) return;
  AEGIS_CHECK_CUDA(cudaEventRecord(comm_marks.back().end, c.comm));
}

// Gather-mode activation: the m ranks of the token group each computed their
// own part of its lanes; one all-gather on the comm stream fills the rest.
// Issued at the matmul's first read (the r = 0 PMult), waited on at once.
void Executor::allgather(u32 x) {
  gather_src[x] = 0;
  const ShardPlan& P = *o.shard;
  Bundle& X = *buf[x];
  const u32 c_in = gather_cin[x];
  if (c_in % P.m) throw Error(AEGIS_EINVAL, "PCMM inputs do not split evenly over the ranks of a token group");
  const size_t words_per_lane = (size_t)X.comps * X.level * c.n;
  const size_t share = (size_t)(c_in / P.m) * words_per_lane;
  cudaEvent_t ready, done;
  AEGIS_CHECK_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  AEGIS_CHECK_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  events.push_back(ready);
  events.push_back(done);
  AEGIS_CHECK_CUDA(cudaEventRecord(ready, c.stream));
  AEGIS_CHECK_CUDA(cudaStreamWaitEvent(c.comm, ready, 0));
  if (o.fault != 1) {
    comm_mark_begin(x);
    p2p_allgather(*o.p2p, X.view().limb(gather_lane0[x] + P.tg_lo * c_in, 0, 0, c.n), share, c.comm);
    comm_mark_end();
    c.count(4);
    comm_bytes += (size_t)(P.m - 1) * share * 8;
  }
  AEGIS_CHECK_CUDA(cudaEventRecord(done, c.comm));
  AEGIS_CHECK_CUDA(cudaStreamWaitEvent(c.stream, done, 0));
}

void Executor::wait_pending(u32 b, u32 lo, u32 hi) {
  std::vector<Pending>& v = pending[b];
  for (size_t k = 0; k < v.size();) {
    if (v[k].lo < hi && lo < v[k].hi) {
      AEGIS_CHECK_CUDA(cudaStreamWaitEvent(c.stream, v[k].ev, 0));
      v.erase(v.begin() + (long)k);
    } else {
      ++k;
    }
  }
}

void Executor::retire(u32 id) {
  if (shadow[id]) materialize(id);
  if (!pending[id].empty()) wait_pending(id);
  if (!buf[id]) return;
  if (donated[id]) {  // storage now belongs to the op's output bundle
    buf[id] = nullptr;
    return;
  }
  if (partial[id]) reduce_partial(id);
  const Bundle& b = *buf[id];
  const hp::CtBundle& cb = g.bundles[id];
  std::vector<std::pair<u32, u32>> runs =
      o.shard ? o.shard->runs(id, 0, cb.lanes) : std::vector<std::pair<u32, u32>>{{0, cb.lanes}};
  if (id == final_bundle && o.host_out) {
    // first 2 comps of every owned lane: host layout [lane][2][level][N]
    const size_t lane_words = (size_t)2 * cb.level * c.n;
    for (auto [s, e] : runs) {
      AEGIS_CHECK_CUDA(cudaMemcpy2DAsync(o.host_out + (size_t)s * lane_words, lane_words * 8,
                                         b.view().limb(s, 0, 0, c.n), (size_t)b.comps * b.level * c.n * 8,
                                         lane_words * 8, e - s, cudaMemcpyDeviceToHost, c.stream));
      d2h_bytes += (size_t)(e - s) * lane_words * 8;
    }
  }
  if (o.d_hash && !is_weight[id]) hash_bundle(id, b);
  c.free_bundle(buf[id]);
  buf[id] = nullptr;
}

// DESIGN.md §2.4 content hash of the lanes this rank owns (or, with
// hash_lanes, of that plan's lanes only) into o.d_hash[id]
void Executor::hash_bundle(u32 id, const Bundle& b) {
  if (!pending[id].empty()) wait_pending(id);
  const u32 lanes = g.bundles[id].lanes;
  const ShardPlan* hp_ = o.hash_lanes ? o.hash_lanes : o.shard;
  std::vector<std::pair<u32, u32>> runs =
      hp_ ? hp_->runs(id, 0, lanes) : std::vector<std::pair<u32, u32>>{{0, lanes}};
  for (auto [a, e] : runs) {
    AEGIS_CHECK_CUDA(launch_hash(b.view(), a, e - a, cur_comps[id], g.bundles[id].level, c.n, o.d_hash + id,
                                 c.stream));
    c.count();
  }
}

// ---------------------------------------------------------------------------
void Executor::find_hoist_groups() {
  group_of.assign(g.ops.size(), -1);
  std::map<u32, int> open;  // src bundle -> open group
  for (size_t i = 0; i < g.ops.size(); ++i) {
    const hp::HeOp& op = g.ops[i];
    if (op.kind == hp::HeOpKind::kRot) {
      const hp::LaneSlice& s = op.ins[0];
      auto it = open.find(s.bundle);
      if (it != open.end()) {
        const Group& gr = groups[it->second];
        if (gr.lane0 != s.lane || gr.count != s.lane_count || gr.level != op.use_level) open.erase(it);
      }
      it = open.find(s.bundle);
      if (it == open.end()) {
        Group ng;
        ng.src = s.bundle;
        ng.lane0 = s.lane;
        ng.count = s.lane_count;
        ng.level = op.use_level;
        groups.push_back(ng);
        it = open.emplace(s.bundle, (int)groups.size() - 1).first;
      }
      Group& gr = groups[it->second];
      gr.last = (int64_t)i;
      ++gr.size;
      group_of[i] = it->second;
    }
    if (op.kind != hp::HeOpKind::kEncode) open.erase(op.out.bundle);  // the source is overwritten
  }
}

// Memory the hoisted ModUp may use: leave room for the rotation outputs, the
// keys and the key-switch workspace.
size_t Executor::hoist_budget(size_t out_bytes) {
  size_t fr = 0, total = 0;
  cudaMemGetInfo(&fr, &total);
  // live bundles (this op's output included: it is allocated before the group
  // is prepared), keys and tables are resident; keep 6 GB for the CUDA/NCCL
  // runtime and 8 GB (or one more output, if larger) for the products,
  // accumulators and key-switch workspaces of the ops inside the group
  const size_t reserved = c.live_bytes + c.total_key_bytes() + ((size_t)c.n * 4 * 16 * kNumExt);
  const size_t cap = total > ((size_t)6 << 30) ? total - ((size_t)6 << 30) : 0;
  const size_t margin = std::max<size_t>((size_t)8 << 30, out_bytes / 4);
  return cap > reserved + margin ? cap - reserved - margin : 0;
}

void Executor::rot_run(const hp::HeOp& op, int64_t i, u32 pos, u32 len) {
  if (full_tg[op.out.bundle] && gather_src[op.ins[0].bundle]) allgather(op.ins[0].bundle);
  Bundle& in = input(op.ins[0]);
  Bundle& out = get(op.out.bundle);
  const u32 L = op.use_level;
  const int gi = group_of[i];
  const u32 src0 = op.ins[0].lane + pos;  // Rot reads lane l of the source for output lane l
  if (!o.hoist || gi < 0 || groups[gi].size < 2 || op.ins[0].lane_count != op.out.lane_count) {
    c.op_rot(out, op.out.lane + pos, in, LaneMap{src0, len}, len, L, op.rot_offset);
    return;
  }
  Group& gr = groups[gi];
  const size_t per_lane = c.modup_words_per_lane(L);
  if (!gr.prepared) {
    gr.prepared = true;
    gr.runs = o.shard ? (full_tg[gr.src] ? o.shard->tg_runs(gr.src, gr.lane0, gr.count)
                                         : o.shard->runs(gr.src, gr.lane0, gr.count))
                      : std::vector<std::pair<u32, u32>>{{gr.lane0, gr.lane0 + gr.count}};
    if (o.dce && !gr.src_live.empty()) {  // only the source lanes some live rotation output needs
      std::vector<std::pair<u32, u32>> lr;
      for (auto [a, e] : gr.runs)
        for (u32 x = a; x < e;) {
          while (x < e && !gr.src_live[x - gr.lane0]) ++x;
          u32 y = x;
          while (y < e && gr.src_live[y - gr.lane0]) ++y;
          if (x < y) lr.emplace_back(x, y);
          x = y;
        }
      gr.runs = lr;
    }
    u32 total = 0;
    for (auto [s, e] : gr.runs) {
      gr.run_off.push_back(total);
      total += e - s;
    }
    gr.hoisted = (u32)std::min<size_t>(total, hoist_budget(out.bytes) / (per_lane * 8));
    if (std::getenv("AEGIS_DEBUG"))
      fprintf(stderr, "[aegis] hoist %s: %u of %u lanes at level %u (%zu MiB/lane, %u rotations)\n",
              g.bundles[gr.src].tag.c_str(), gr.hoisted, total, L, per_lane * 8 >> 20, gr.size);
    if (gr.hoisted > 0) {
      gr.ext = c.alloc(per_lane * gr.hoisted);
      const size_t in_ls = (size_t)in.comps * in.level * c.n;
      for (size_t r = 0; r < gr.runs.size(); ++r) {
        const u32 off = gr.run_off[r];
        if (off >= gr.hoisted) break;
        const u32 cnt = std::min(gr.runs[r].second - gr.runs[r].first, gr.hoisted - off);
        c.modup(in.view().limb(gr.runs[r].first, 1, 0, c.n), in_ls, cnt, L, gr.ext + (size_t)off * per_lane);
      }
    }
  }
  // locate [src0, src0+len) in the compact (run-ordered) ext buffer
  u32 done = 0;
  while (done < len) {
    const u32 lane = src0 + done;
    size_t r = 0;
    while (r < gr.runs.size() && !(lane >= gr.runs[r].first && lane < gr.runs[r].second)) ++r;
    if (r == gr.runs.size()) throw Error(AEGIS_ELOGIC, "rotation of a lane this rank does not own");
    const u32 idx = gr.run_off[r] + (lane - gr.runs[r].first);
    u32 cnt = std::min(len - done, gr.runs[r].second - lane);
    if (idx < gr.hoisted) {
      cnt = std::min(cnt, gr.hoisted - idx);
      c.op_rot_cached(out, op.out.lane + pos + done, in, LaneMap{lane, cnt}, cnt, L, op.rot_offset,
                      gr.ext + (size_t)idx * per_lane);
    } else {
      c.op_rot(out, op.out.lane + pos + done, in, LaneMap{lane, cnt}, cnt, L, op.rot_offset);
    }
    done += cnt;
  }
}

// ---------------------------------------------------------------------------
std::vector<std::pair<u32, u32>> Executor::out_runs(const hp::HeOp& op) const {
  const u32 n = op.out.lane_count;
  std::vector<std::pair<u32, u32>> r;
  if (!o.shard) {
    r.emplace_back(0, n);
  } else if (full_tg[op.out.bundle]) {  // gather-mode rotations: every lane of the token group
    for (auto [s, e] : o.shard->tg_runs(op.out.bundle, op.out.lane, n)) r.emplace_back(s - op.out.lane, e - op.out.lane);
  } else {
    for (auto [s, e] : o.shard->runs(op.out.bundle, op.out.lane, n)) r.emplace_back(s - op.out.lane, e - op.out.lane);
  }
  if (!o.dce) return r;
  std::vector<std::pair<u32, u32>> lr;  // dead-lane elimination: live output positions only
  const std::vector<char>& lv = live[op.out.bundle];
  for (auto [a, e] : r)
    for (u32 x = a; x < e;) {
      while (x < e && !lv[op.out.lane + x]) ++x;
      u32 y = x;
      while (y < e && lv[op.out.lane + y]) ++y;
      if (x < y) lr.emplace_back(x, y);
      x = y;
    }
  return lr;
}

// first position >= pos where a wrapped operand (count != n) wraps around
u32 Executor::wrap_end(const hp::HeOp& op, u32 pos, u32 end) const {
  const u32 n = op.out.lane_count;
  for (const hp::LaneSlice& s : op.ins)
    if (s.lane_count != n && s.lane_count) end = std::min(end, (pos / s.lane_count + 1) * s.lane_count);
  return end;
}

LaneMap Executor::sub_map(const hp::LaneSlice& s, u32 n, u32 pos, u32 len) {
  return s.lane_count == n ? LaneMap{s.lane + pos, len} : LaneMap{s.lane + pos % s.lane_count, len};
}

void Executor::pmult(const hp::HeOp& op, int64_t i) {
  if (!op.accumulate || op.ins.size() != 2) throw Error(AEGIS_ELOGIC, "unsupported PMult form");
  if (gather_acc[op.out.bundle] && gather_src[op.ins[0].bundle]) allgather(op.ins[0].bundle);
  Bundle& x = input(op.ins[0]);
  Bundle& acc = get(op.out.bundle);
  const u32 chunk = g.bundles[op.out.bundle].chunk_period;
  const u32 L = op.use_level;
  const Bundle* ws = o.stored_weights ? &input(op.ins[1]) : nullptr;
  const u32 wl0 = op.ins[1].lane;
  if (!o.shard) {
    c.op_pmult(acc, op.out.lane, op.out.lane_count, chunk, x, op.ins[0].lane, op.ins[0].lane_count, op.ins[1].bundle,
               op.ins[1].lane_count, L, 0, ~0u, 0, ~0u, ws, wl0);
    return;
  }
  const ShardPlan& P = *o.shard;
  if (P.m > 1 && gather_acc[op.out.bundle]) {
    // output-stationary: all inputs of the group, this rank's share of every sub-tensor
    const PcmmShape sh = pcmm_shape(op.ins[0].lane_count, op.out.lane_count, op.ins[1].lane_count, chunk);
    const u32 share = sh.c_sub / P.m;
    c.op_pmult(acc, op.out.lane, op.out.lane_count, chunk, x, op.ins[0].lane, op.ins[0].lane_count, op.ins[1].bundle,
               op.ins[1].lane_count, L, P.tg_lo, P.tg_lo + 1, 0, ~0u, ws, wl0, P.part * share, share);
    return;
  }
  if (P.m == 1) {
    c.op_pmult(acc, op.out.lane, op.out.lane_count, chunk, x, op.ins[0].lane, op.ins[0].lane_count, op.ins[1].bundle,
               op.ins[1].lane_count, L, P.tg_lo, P.tg_hi, 0, ~0u, ws, wl0);
    return;
  }
  // input-stationary: this rank's input positions into every output of its group
  const PcmmShape sh = pcmm_shape(op.ins[0].lane_count, op.out.lane_count, op.ins[1].lane_count, chunk);
  const u32 t = P.tg_lo;
  u32 ci_lo = sh.c_in, ci_hi = 0;
  for (u32 ci = 0; ci < sh.c_in; ++ci)
    if (P.owns(op.ins[0].bundle, op.ins[0].lane + t * sh.c_in + ci)) {
      ci_lo = std::min(ci_lo, ci);
      ci_hi = std::max(ci_hi, ci + 1);
    }
  if (ci_lo < ci_hi)
    c.op_pmult(acc, op.out.lane, op.out.lane_count, chunk, x, op.ins[0].lane, op.ins[0].lane_count, op.ins[1].bundle,
               op.ins[1].lane_count, L, t, t + 1, ci_lo, ci_hi, ws, wl0);
  partial[op.out.bundle] = 1;
  // the accumulator is complete on this rank: start its exchange now, on the comm stream
  if (o.p2p && last_pmult[op.out.bundle] == i) reduce_async(op.out.bundle);
}

// Device-synchronised form of reduce_partial: one p2p_exchange per sub-tensor
// on the comm stream, started right after the last PMult of the accumulator;
// the compute stream waits (cudaStreamWaitEvent) only when an op touches the
// sub-tensor's lanes, so the rescale of sub-tensor s overlaps the exchange of
// sub-tensor s + 1.
void Executor::reduce_async(u32 b) {
  partial[b] = 0;
  const ShardPlan& P = *o.shard;
  Bundle& acc = *buf[b];
  const hp::HeOp& pm = g.ops[last_pmult[b]];
  const PcmmShape sh = pcmm_shape(pm.ins[0].lane_count, pm.out.lane_count, pm.ins[1].lane_count,
                                  g.bundles[b].chunk_period);
  if (sh.c_sub % P.m) throw Error(AEGIS_EINVAL, "PCMM outputs do not split evenly over the ranks of a token group");
  const u32 t = P.tg_lo, share = sh.c_sub / P.m;
  const uint64_t words_per_lane = (uint64_t)acc.comps * acc.level * c.n;
  cudaEvent_t ready;
  AEGIS_CHECK_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  events.push_back(ready);
  AEGIS_CHECK_CUDA(cudaEventRecord(ready, c.stream));
  AEGIS_CHECK_CUDA(cudaStreamWaitEvent(c.comm, ready, 0));
  for (u32 s = 0; s < sh.S; ++s) {
    const u32 lane0 = pm.out.lane + pcmm_lane(sh, t, s * sh.c_sub);
    if (o.fault != 1) {
      comm_mark_begin(b);
      p2p_exchange(*o.p2p, acc.view().limb(lane0, 0, 0, c.n), words_per_lane * share, c.comm);
      comm_mark_end();
      c.count(4);
      comm_bytes += (size_t)(P.m - 1) * words_per_lane * share * 8;
    }
    const u32 mine = lane0 + P.part * share;
    AEGIS_CHECK_CUDA(launch_reduce_lanes(acc.view(), mine, share, acc.comps, acc.level, c.n, c.d_pc, c.comm));
    c.count();
    cudaEvent_t done;
    AEGIS_CHECK_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    events.push_back(done);
    AEGIS_CHECK_CUDA(cudaEventRecord(done, c.comm));
    pending[b].push_back(Pending{mine, mine + share, done});
  }
}

// Sum the partial accumulators of this rank's token group over its m ranks
// (one reduce-scatter per sub-tensor) and canonicalise the owned share.
void Executor::reduce_partial(u32 b) {
  partial[b] = 0;
  if (!o.shard || o.shard->m == 1) return;
  if (!o.reduce && o.fault != 1)
    throw Error(AEGIS_ELOGIC, "sharded PCMM needs a reduce-scatter hook (aegis_graph_set_reducer) or a p2p window");
  const ShardPlan& P = *o.shard;
  Bundle& acc = *buf[b];
  // find the PCMM shape from the last PMult writing this bundle
  const hp::HeOp* pm = nullptr;
  for (const hp::HeOp& op : g.ops)
    if (op.kind == hp::HeOpKind::kPMult && op.out.bundle == b) pm = &op;
  if (!pm) throw Error(AEGIS_ELOGIC, "partial bundle without a PCMM writer");
  const PcmmShape sh = pcmm_shape(pm->ins[0].lane_count, pm->out.lane_count, pm->ins[1].lane_count,
                                  g.bundles[b].chunk_period);
  if (sh.c_sub % P.m) throw Error(AEGIS_EINVAL, "PCMM outputs do not split evenly over the ranks of a token group");
  const u32 t = P.tg_lo, share = sh.c_sub / P.m;
  const uint64_t words_per_lane = (uint64_t)acc.comps * acc.level * c.n;
  AEGIS_CHECK_CUDA(cudaStreamSynchronize(c.stream));
  for (u32 s = 0; s < sh.S; ++s) {
    const u32 lane0 = pm->out.lane + pcmm_lane(sh, t, s * sh.c_sub);
    u64* base = acc.view().limb(lane0, 0, 0, c.n);
    if (o.fault != 1) {
      if (o.reduce(o.reduce_user, base, words_per_lane * share, t) != 0)
        throw Error(AEGIS_ENCCL, "reduce-scatter hook failed");
      comm_bytes += (size_t)(P.m - 1) * words_per_lane * share * 8;
    }
    AEGIS_CHECK_CUDA(launch_reduce_lanes(acc.view(), lane0 + P.part * share, share, acc.comps, acc.level, c.n, c.d_pc,
                                         c.stream));
    c.count();
  }
}

// Buffer donation: an element-wise op (Rescale, non-accumulating CAdd) whose
// first operand dies here and covers the output lane-for-lane writes its result
// into the operand's storage (same strides, fewer limbs used).  Both kernels
// read each position before writing it, so in-place is exact; it removes the
// 53 GB score copy at T = 2048.
void Executor::donate(const hp::HeOp& op, int64_t i) {
  using K = hp::HeOpKind;
  if (op.kind != K::kRescale && !(op.kind == K::kCAdd && !op.accumulate)) return;
  if (buf[op.out.bundle] || op.ins.empty()) return;
  const hp::LaneSlice& s = op.ins[0];
  if (s.bundle == op.out.bundle || last_use[s.bundle] != i || !buf[s.bundle]) return;
  const hp::CtBundle& ob = g.bundles[op.out.bundle];
  Bundle& in = *buf[s.bundle];
  if (s.lane != 0 || op.out.lane != 0 || s.lane_count != ob.lanes || op.out.lane_count != ob.lanes ||
      in.lanes != ob.lanes || in.level < ob.level || in.level > ob.level + 1 ||
      in.comps != std::max<u32>(2, alloc_comps[op.out.bundle]))
    return;  // only when the donated storage is (nearly) the output's own size
  for (size_t k = 1; k < op.ins.size(); ++k)  // a second operand must not alias differently
    if (op.ins[k].bundle == s.bundle && (op.ins[k].lane != 0 || op.ins[k].lane_count != ob.lanes)) return;
  if (partial[s.bundle]) reduce_partial(s.bundle);
  if (o.d_hash) hash_bundle(s.bundle, in);  // the operand dies now: hash it before it is overwritten
  buf[op.out.bundle] = buf[s.bundle];  // same allocation, operand strides
  donated[s.bundle] = 1;               // still readable by this op; never freed or hashed again
  cur_comps[op.out.bundle] = 2;
}

// Wrapped accumulation (score.acc at T = 2048: 64 CAdds each adding a 48-lane
// product into all 1,536 lanes, acc[j] += prod[j mod 48]).  Modular addition
// is exact and associative, so the addends are summed at the operand's width,
// S += prod (48 lanes), and the bundle is updated once, acc[j] += S[j mod 48],
// before anything else touches it.  Every bundle any op reads is bit-identical
// to the op-by-op order; the 64 full-width read-modify-writes (~160 GB each
// way in total per op) become 64 narrow ones plus one wide one.
bool Executor::wrap_deferrable(const hp::HeOp& op) const {
  if (!o.wrap_defer || o.dce || op.kind != hp::HeOpKind::kCAdd || !op.accumulate || op.ins.size() != 1)
    return false;
  const hp::LaneSlice& s = op.ins[0];
  const u32 n = g.bundles[op.out.bundle].lanes, m = s.lane_count;
  if (s.bundle == op.out.bundle || op.out.lane != 0 || op.out.lane_count != n || !m || m >= n || n % m) return false;
  const Bundle* sh = shadow[op.out.bundle];
  return !sh || (sh->lanes == m && shadow_level[op.out.bundle] == op.use_level);
}

void Executor::materialize(u32 b) {
  Bundle* S = shadow[b];
  shadow[b] = nullptr;
  Bundle& X = get(b);
  const u32 lanes = g.bundles[b].lanes, m = S->lanes;
  if (!o.shard) {
    c.op_cadd(X, 0, lanes, *S, LaneMap{0, m}, nullptr, LaneMap{0, 1}, shadow_level[b], true);
  } else {  // owned lanes only, split where the operand index j mod m wraps
    for (auto [rs, re] : o.shard->runs(b, 0, lanes))
      for (u32 pos = rs; pos < re;) {
        const u32 end = std::min(re, (pos / m + 1) * m);
        c.op_cadd(X, pos, end - pos, *S, LaneMap{pos % m, end - pos}, nullptr, LaneMap{0, 1}, shadow_level[b], true);
        pos = end;
      }
  }
  c.free_bundle(S);
  cur_comps[b] = 2;
}

void Executor::step(const hp::HeOp& op, int64_t i) {
  using K = hp::HeOpKind;
  const u32 L = op.use_level;
  if (op.kind == K::kEncode) {
    if (!o.stored_weights) return;  // weights are generated inside the PMult kernel (kGenerate)
    Bundle& w = get(op.out.bundle);  // stored form: the kGenerate rows land in HBM
    AEGIS_CHECK_CUDA(launch_limb_generate(w.view(), 0, w.lanes, 1, 0, w.level, c.n, c.seed_weight, 2,
                                          op.out.bundle, c.d_pc, c.stream));
    c.count();
    cur_comps[op.out.bundle] = 1;
    return;
  }
  for (const hp::LaneSlice& s : op.ins)
    if (shadow[s.bundle]) materialize(s.bundle);
  const bool defer = wrap_deferrable(op);
  if (shadow[op.out.bundle] && !defer) materialize(op.out.bundle);
  if (defer) {
    const hp::LaneSlice& s = op.ins[0];
    Bundle& in = input(s);
    Bundle*& S = shadow[op.out.bundle];
    if (!S) {
      S = c.new_bundle(s.lane_count, 2, L, true);
      shadow_level[op.out.bundle] = L;
    }
    if (!o.shard) {
      c.op_cadd(*S, 0, s.lane_count, in, LaneMap{s.lane, s.lane_count}, nullptr, LaneMap{0, 1}, L, true);
    } else {  // the operand lanes this rank owns (the only ones its output lanes read)
      for (auto [rs, re] : o.shard->runs(s.bundle, s.lane, s.lane_count))
        c.op_cadd(*S, rs - s.lane, re - rs, in, LaneMap{rs, re - rs}, nullptr, LaneMap{0, 1}, L, true);
    }
    get(op.out.bundle);  // the bundle exists from here on, as if written
    cur_comps[op.out.bundle] = 2;
    return;
  }
  if (op.kind == K::kPAdd) throw Error(AEGIS_ELOGIC, "PAdd is not emitted by the reference lowering");
  if (op.kind == K::kPMult) {
    pmult(op, i);
    cur_comps[op.out.bundle] = 2;
    return;
  }
  if (partial[op.out.bundle]) reduce_partial(op.out.bundle);
  donate(op, i);
  const u32 n = op.out.lane_count;
  for (auto [rs, re] : out_runs(op)) {
    for (u32 pos = rs; pos < re;) {
      const u32 end = wrap_end(op, pos, re);
      const u32 len = end - pos;
      switch (op.kind) {
        case K::kRot:
          rot_run(op, i, pos, len);
          break;
        case K::kRelin:
          c.op_relin(get(op.out.bundle), op.out.lane + pos, len, L);
          break;
        case K::kRescale: {
          // only the exchanges covering these lanes (the rest may still be in flight)
          const LaneMap im = sub_map(op.ins[0], n, pos, len);
          Bundle& in = im.count == len ? input(op.ins[0], im.lane0, im.lane0 + len) : input(op.ins[0]);
          c.op_rescale(get(op.out.bundle), op.out.lane + pos, in, sub_map(op.ins[0], n, pos, len), len, L);
          break;
        }
        case K::kBoot: {
          if (gather_src[op.ins[0].bundle] && full_tg[op.out.bundle]) allgather(op.ins[0].bundle);
          Bundle& in = input(op.ins[0]);
          c.op_boot(get(op.out.bundle), op.out.lane + pos, in, sub_map(op.ins[0], n, pos, len), len, L,
                    g.bundles[op.out.bundle].level);
          break;
        }
        case K::kCMult: {
          Bundle& a = input(op.ins[0]);
          Bundle& b = input(op.ins[1]);
          c.op_cmult(get(op.out.bundle), op.out.lane + pos, len, a, sub_map(op.ins[0], n, pos, len), b,
                     sub_map(op.ins[1], n, pos, len), L);
          break;
        }
        case K::kCAdd: {
          Bundle& a = input(op.ins[0]);
          Bundle* b = op.ins.size() > 1 ? &input(op.ins[1]) : nullptr;
          c.op_cadd(get(op.out.bundle), op.out.lane + pos, len, a, sub_map(op.ins[0], n, pos, len), b,
                    b ? sub_map(op.ins[1], n, pos, len) : LaneMap{0, 1}, L, op.accumulate);
          break;
        }
        default:
          throw Error(AEGIS_ELOGIC, "unknown op kind");
      }
      pos = end;
    }
  }
  // a rank that owns no output lane of this op still materialises the bundle
  // so later readers find it (its lanes are never touched)
  get(op.out.bundle);
  cur_comps[op.out.bundle] = op.kind == K::kCMult ? 3 : 2;
  if (op.kind == K::kRot && group_of[i] >= 0) {
    Group& gr = groups[group_of[i]];
    if (gr.last == i && gr.ext) {
      c.release(gr.ext);
      gr.ext = nullptr;
    }
  }
}

void Executor::run() {
  // graph inputs: synthetic (PRNG tag 1) or copied from host memory
  size_t off = 0;
  for (u32 in : g.graph_inputs) {
    Bundle& b = get(in);
    const size_t lane_words = (size_t)2 * b.level * c.n;
    std::vector<std::pair<u32, u32>> runs =
        o.shard ? o.shard->runs(in, 0, b.lanes) : std::vector<std::pair<u32, u32>>{{0, b.lanes}};
    if (o.host_in) {
      for (auto [s, e] : runs) {
        AEGIS_CHECK_CUDA(cudaMemcpy2DAsync(b.view().limb(s, 0, 0, c.n), (size_t)b.comps * b.level * c.n * 8,
                                           o.host_in + off + (size_t)s * lane_words, lane_words * 8, lane_words * 8,
                                           e - s, cudaMemcpyHostToDevice, c.stream));
        h2d_bytes += (size_t)(e - s) * lane_words * 8;
      }
      off += (size_t)b.lanes * lane_words;
    } else {
      AEGIS_CHECK_CUDA(launch_fill_uniform(b.view(), b.lanes, 2, b.level, c.n, c.seed_input, 1, in, c.d_ident, c.d_pc,
                                           c.stream));
      c.count();
    }
  }
  if (o.host_out && !g.ops.empty()) final_bundle = g.ops.back().out.bundle;
  const int64_t nops = o.max_ops < 0 ? (int64_t)g.ops.size() : std::min<int64_t>(o.max_ops, (int64_t)g.ops.size());
  std::vector<cudaEvent_t> ev;
  if (o.op_ms) {
    ev.resize(nops + 1);
    for (auto& e : ev) AEGIS_CHECK_CUDA(cudaEventCreate(&e));
    AEGIS_CHECK_CUDA(cudaEventRecord(ev[0], c.stream));
  }
  for (int64_t i = 0; i < nops; ++i) {
    const hp::HeOp& op = g.ops[i];
    try {
      step(op, i);
      if (o.op_ms) AEGIS_CHECK_CUDA(cudaEventRecord(ev[i + 1], c.stream));
    } catch (const Error& e) {
      std::string live;
      if (e.code == AEGIS_EOOM) {  // what is holding the memory
        std::vector<std::pair<size_t, u32>> v;
        for (u32 b = 0; b < buf.size(); ++b)
          if (buf[b] && !donated[b]) v.emplace_back(buf[b]->bytes, b);
        std::sort(v.rbegin(), v.rend());
        live = " live:";
        for (size_t k = 0; k < v.size() && k < 6; ++k)
          live += " " + g.bundles[v[k].second].tag + "=" + std::to_string(v[k].first >> 20) + "MiB";
        size_t hoisted = 0;
        for (auto& gr : groups)
          if (gr.ext) hoisted += (size_t)gr.hoisted * c.modup_words_per_lane(gr.level) * 8;
        live += " hoisted=" + std::to_string(hoisted >> 20) + "MiB";
      }
      throw Error(e.code, std::string(e.what()) + " [op " + std::to_string(i) + " -> " +
                              g.bundles[op.out.bundle].tag + "]" + live);
    }
    std::set<u32> touched{op.out.bundle};
    for (auto& s : op.ins) touched.insert(s.bundle);
    for (u32 b : touched)
      if (last_use[b] == i && i + 1 < (int64_t)g.ops.size()) retire(b);
  }
  for (u32 b = 0; b < buf.size(); ++b) retire(b);
  for (auto& gr : groups)
    if (gr.ext) {
      c.release(gr.ext);
      gr.ext = nullptr;
    }
  if (o.op_ms) {
    AEGIS_CHECK_CUDA(cudaStreamSynchronize(c.stream));
    AEGIS_CHECK_CUDA(cudaStreamSynchronize(c.comm));
    o.op_ms->assign(nops, 0.0f);
    for (int64_t i = 0; i < nops; ++i) cudaEventElapsedTime(&(*o.op_ms)[i], ev[i], ev[i + 1]);
    if (o.comm_trace) {
      o.comm_trace->clear();
      for (const CommMark& m : comm_marks) {
        float s0 = 0, s1 = 0;
        cudaEventElapsedTime(&s0, ev[0], m.start);
        cudaEventElapsedTime(&s1, ev[0], m.end);
        o.comm_trace->insert(o.comm_trace->end(), {s0, s1, (float)m.bundle});
        cudaEventDestroy(m.start);
        cudaEventDestroy(m.end);
      }
      comm_marks.clear();
    }
    for (auto& e : ev) cudaEventDestroy(e);
  }
}

}  // namespace aegis

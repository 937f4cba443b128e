// capi.cu -- the extern "C" boundary of libaegis (include/aegis.h) and the
// HE-graph executor (SPEC.md:407-415 exec_sequential, run on one B200).
//
// No exception crosses the boundary: every entry point catches and maps to an
// AEGIS_E* code, keeping the message for aegis_last_error().
#include <algorithm>
#include <cstring>
#include <fstream>
#include <set>
#include <sstream>

#include "context.h"
#include "heplan_ir.h"

using aegis::Bundle;
using aegis::Context;
using aegis::Error;
using aegis::LaneMap;
using aegis::u32;
using aegis::u64;
namespace hp = aegis::heplan;

struct aegis_ctx {
  std::unique_ptr<Context> c;
  std::string err;
};
struct aegis_bundle {
  Bundle* b = nullptr;
};

namespace {

thread_local std::string g_create_err;

template <class F>
int guard(aegis_ctx* ctx, F&& f) {
  try {
    f();
    return AEGIS_OK;
  } catch (const Error& e) {
    if (ctx) ctx->err = e.what();
    return e.code;
  } catch (const std::invalid_argument& e) {
    if (ctx) ctx->err = e.what();
    return AEGIS_EINVAL;
  } catch (const std::logic_error& e) {
    if (ctx) ctx->err = e.what();
    return AEGIS_ELOGIC;
  } catch (const std::bad_alloc& e) {
    if (ctx) ctx->err = "host allocation failed";
    return AEGIS_EOOM;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    return AEGIS_ECUDA;
  }
}

Bundle& need(aegis_bundle* b) {
  if (!b || !b->b) throw Error(AEGIS_EINVAL, "null bundle");
  return *b->b;
}
const Bundle& need(const aegis_bundle* b) {
  if (!b || !b->b) throw Error(AEGIS_EINVAL, "null bundle");
  return *b->b;
}
void check_lanes(const Bundle& b, u32 lane, u32 count, const char* what) {
  if ((uint64_t)lane + count > b.lanes) throw Error(AEGIS_EINVAL, std::string(what) + ": lane range out of bounds");
}
void check_level(const Bundle& b, u32 level, const char* what) {
  if (level == 0) throw Error(AEGIS_EINVAL, "exhausted modulus chain");  // ckks.hpp:149
  if (level > b.level) throw Error(AEGIS_EINVAL, std::string(what) + ": level exceeds bundle level");
}

}  // namespace

// ===========================================================================
// Graph executor
// ===========================================================================
struct aegis_graph {
  hp::HeOpGraph g;
  std::string header;
  uint64_t peak = 0;
  u32 shard_lo = 0, shard_hi = 0xffffffffu;
};

namespace {

struct Exec {
  Context& c;
  const hp::HeOpGraph& g;
  std::vector<Bundle*> buf;
  std::vector<u32> alloc_comps, cur_comps;
  std::vector<char> zero_first;
  std::vector<int64_t> last_use;
  unsigned long long* d_hash = nullptr;

  Exec(Context& ctx, const hp::HeOpGraph& graph) : c(ctx), g(graph) {
    const size_t nb = g.bundles.size();
    buf.assign(nb, nullptr);
    alloc_comps.resize(nb);
    cur_comps.assign(nb, 0);
    zero_first.assign(nb, 0);
    last_use.assign(nb, -1);
    std::vector<char> seen(nb, 0);
    for (size_t i = 0; i < nb; ++i) alloc_comps[i] = g.bundles[i].components;
    for (size_t i = 0; i < g.ops.size(); ++i) {
      const hp::HeOp& op = g.ops[i];
      last_use[op.out.bundle] = (int64_t)i;
      for (auto& s : op.ins) last_use[s.bundle] = (int64_t)i;
      if (op.kind == hp::HeOpKind::kCMult) alloc_comps[op.out.bundle] = 3;
      if (!seen[op.out.bundle] && op.kind != hp::HeOpKind::kEncode) {
        seen[op.out.bundle] = 1;
        zero_first[op.out.bundle] = op.accumulate ? 1 : 0;
      }
    }
    find_hoist_groups();
  }

  // ---- hoisted ModUp across rotations of one source ----------
  // A group is a run of Rot ops reading the same (bundle, lanes, level) with no
  // write to that bundle in between (the 63 diagonals of a PCMM / CCMM).
  struct Group {
    u32 src, lane0, count, level;
    int64_t last = -1;
    u32 size = 0;
    u64* ext = nullptr;
    u32 hoisted_lanes = 0;
    bool prepared = false;
  };
  std::vector<Group> groups;
  std::vector<int> group_of;  // per op (-1 = none)

  void find_hoist_groups() {
    group_of.assign(g.ops.size(), -1);
    std::map<u32, int> open;  // src bundle -> open group
    for (size_t i = 0; i < g.ops.size(); ++i) {
      const hp::HeOp& op = g.ops[i];
      if (op.kind == hp::HeOpKind::kRot) {
        const hp::LaneSlice& s = op.ins[0];
        auto it = open.find(s.bundle);
        if (it != open.end()) {
          Group& gr = groups[it->second];
          if (gr.lane0 != s.lane || gr.count != s.lane_count || gr.level != op.use_level) open.erase(it);
        }
        it = open.find(s.bundle);
        if (it == open.end()) {
          groups.push_back(Group{s.bundle, s.lane, s.lane_count, op.use_level});
          it = open.emplace(s.bundle, (int)groups.size() - 1).first;
        }
        Group& gr = groups[it->second];
        gr.last = (int64_t)i;
        ++gr.size;
        group_of[i] = it->second;
      }
      if (op.kind != hp::HeOpKind::kEncode) open.erase(op.out.bundle);  // the source is being overwritten
    }
  }

  // memory the hoisted ModUp may use: leave room for the rotation outputs and
  // the key-switch workspace
  size_t hoist_budget(size_t out_bytes) {
    size_t fr = 0, total = 0;
    cudaMemGetInfo(&fr, &total);
    const size_t reserved = c.live_bytes + c.total_key_bytes() + ((size_t)c.n * 2 * 16 * aegis::kNumExt);
    const size_t cap = (size_t)(0.92 * (double)total);
    const size_t margin = out_bytes + ((size_t)6 << 30);
    return cap > reserved + margin ? cap - reserved - margin : 0;
  }

  void rot(const hp::HeOp& op, int64_t i, Bundle& in, Bundle& out, u32 lanes, u32 L) {
    const int gi = group_of[i];
    if (gi < 0 || groups[gi].size < 2 || op.ins[0].lane_count != lanes || hoist_disabled) {
      c.op_rot(out, op.out.lane, in, lm(op.ins[0]), lanes, L, op.rot_offset);
      return;
    }
    Group& gr = groups[gi];
    const size_t per_lane = c.modup_words_per_lane(L);
    if (!gr.prepared) {
      gr.prepared = true;
      const size_t budget = hoist_budget(out.bytes);
      gr.hoisted_lanes = (u32)std::min<size_t>(lanes, budget / (per_lane * 8));
      if (gr.hoisted_lanes > 0) {
        gr.ext = c.alloc(per_lane * gr.hoisted_lanes);
        c.modup(in.view().limb(op.ins[0].lane, 1, 0, c.n), (size_t)in.comps * in.level * c.n, gr.hoisted_lanes, L,
                gr.ext);
      }
    }
    const u32 H = gr.hoisted_lanes;
    if (H > 0)
      c.op_rot_cached(out, op.out.lane, in, LaneMap{op.ins[0].lane, H}, H, L, op.rot_offset, gr.ext);
    if (H < lanes)
      c.op_rot(out, op.out.lane + H, in, LaneMap{op.ins[0].lane + H, lanes - H}, lanes - H, L, op.rot_offset);
    if (gr.last == i && gr.ext) {
      c.release(gr.ext);
      gr.ext = nullptr;
    }
  }
  bool hoist_disabled = false;
  int64_t cur_op = 0;

  Bundle& get(u32 id) {
    if (!buf[id]) {
      const hp::CtBundle& cb = g.bundles[id];
      buf[id] = c.new_bundle(cb.lanes, std::max<u32>(2, alloc_comps[id]), cb.level, zero_first[id] != 0);
      cur_comps[id] = 2;
    }
    return *buf[id];
  }
  Bundle& input(const hp::LaneSlice& s) {
    if (!buf[s.bundle]) throw Error(AEGIS_ELOGIC, "op reads bundle " + g.bundles[s.bundle].tag + " before it is written");
    return *buf[s.bundle];
  }
  void retire(u32 id) {
    if (!buf[id]) return;
    if (id == final_bundle && host_out) {
      const Bundle& b = *buf[id];
      // first 2 comps of every lane: [lane][2][level][N]
      AEGIS_CHECK_CUDA(cudaMemcpy2DAsync(host_out, (size_t)2 * b.level * c.n * 8, b.ptr,
                                         (size_t)b.comps * b.level * c.n * 8, (size_t)2 * b.level * c.n * 8,
                                         b.lanes, cudaMemcpyDeviceToHost, c.stream));
    }
    if (d_hash) {
      AEGIS_CHECK_CUDA(aegis::launch_hash(buf[id]->view(), buf[id]->lanes, cur_comps[id], g.bundles[id].level, c.n,
                                          d_hash + id, c.stream));
      c.count();
    }
    c.free_bundle(buf[id]);
    buf[id] = nullptr;
  }

  const u64* host_in = nullptr;  // graph inputs from host memory (end-to-end path)
  u64* host_out = nullptr;       // final bundle to host memory
  u32 final_bundle = 0xffffffffu;

  void run(int64_t max_ops) {
    size_t off = 0;
    for (u32 in : g.graph_inputs) {
      Bundle& b = get(in);
      if (host_in) {
        const size_t words = (size_t)b.lanes * 2 * b.level * c.n;
        AEGIS_CHECK_CUDA(cudaMemcpyAsync(b.ptr, host_in + off, words * 8, cudaMemcpyHostToDevice, c.stream));
        off += words;
      } else {
        AEGIS_CHECK_CUDA(aegis::launch_fill_uniform(b.view(), b.lanes, 2, b.level, c.n, c.seed_input, 1, in,
                                                    c.d_ident, c.d_pc, c.stream));
        c.count();
      }
    }
    if (host_out && !g.ops.empty()) final_bundle = g.ops.back().out.bundle;
    const int64_t nops = max_ops < 0 ? (int64_t)g.ops.size() : std::min<int64_t>(max_ops, (int64_t)g.ops.size());
    for (int64_t i = 0; i < nops; ++i) {
      const hp::HeOp& op = g.ops[i];
      cur_op = i;
      step(op);
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
  }

  static LaneMap lm(const hp::LaneSlice& s) { return LaneMap{s.lane, s.lane_count}; }

  void step(const hp::HeOp& op) {
    const u32 L = op.use_level;
    const u32 lanes = op.out.lane_count;
    switch (op.kind) {
      case hp::HeOpKind::kEncode:
        return;  // weights are generated inside the PMult kernel (kGenerate)
      case hp::HeOpKind::kRot: {
        Bundle& in = input(op.ins[0]);
        Bundle& out = get(op.out.bundle);
        rot(op, cur_op, in, out, lanes, L);
        cur_comps[op.out.bundle] = 2;
        return;
      }
      case hp::HeOpKind::kRelin: {
        Bundle& b = get(op.out.bundle);
        c.op_relin(b, op.out.lane, lanes, L);
        cur_comps[op.out.bundle] = 2;
        return;
      }
      case hp::HeOpKind::kRescale: {
        Bundle& in = input(op.ins[0]);
        Bundle& out = get(op.out.bundle);
        c.op_rescale(out, op.out.lane, in, lm(op.ins[0]), lanes, L);
        cur_comps[op.out.bundle] = 2;
        return;
      }
      case hp::HeOpKind::kBoot: {
        Bundle& in = input(op.ins[0]);
        Bundle& out = get(op.out.bundle);
        c.op_boot(out, op.out.lane, in, lm(op.ins[0]), lanes, L, g.bundles[op.out.bundle].level);
        cur_comps[op.out.bundle] = 2;
        return;
      }
      case hp::HeOpKind::kCMult: {
        Bundle& a = input(op.ins[0]);
        Bundle& b = input(op.ins[1]);
        Bundle& out = get(op.out.bundle);
        c.op_cmult(out, op.out.lane, lanes, a, lm(op.ins[0]), b, lm(op.ins[1]), L);
        cur_comps[op.out.bundle] = 3;
        return;
      }
      case hp::HeOpKind::kCAdd: {
        Bundle& a = input(op.ins[0]);
        Bundle* b = op.ins.size() > 1 ? &input(op.ins[1]) : nullptr;
        Bundle& out = get(op.out.bundle);
        c.op_cadd(out, op.out.lane, lanes, a, lm(op.ins[0]), b, b ? lm(op.ins[1]) : LaneMap{0, 1}, L, op.accumulate);
        cur_comps[op.out.bundle] = 2;
        return;
      }
      case hp::HeOpKind::kPMult: {
        if (!op.accumulate || op.ins.size() != 2) throw Error(AEGIS_ELOGIC, "unsupported PMult form");
        Bundle& x = input(op.ins[0]);
        Bundle& acc = get(op.out.bundle);
        c.op_pmult(acc, op.out.lane, lanes, g.bundles[op.out.bundle].chunk_period, x, op.ins[0].lane,
                   op.ins[0].lane_count, op.ins[1].bundle, op.ins[1].lane_count, L);
        cur_comps[op.out.bundle] = 2;
        return;
      }
      case hp::HeOpKind::kPAdd:
        throw Error(AEGIS_ELOGIC, "PAdd is not emitted by the reference lowering");
    }
  }
};

}  // namespace

// ===========================================================================
extern "C" {

int aegis_ctx_create(const aegis_params* params, int device, aegis_ctx** out) {
  if (!params || !out) return AEGIS_EINVAL;
  *out = nullptr;
  auto* h = new aegis_ctx;
  const int rc = guard(h, [&] { h->c.reset(new Context(*params, device)); });
  if (rc != AEGIS_OK) {
    g_create_err = h->err;
    delete h;
    return rc;
  }
  *out = h;
  return AEGIS_OK;
}

int aegis_ctx_destroy(aegis_ctx* ctx) {
  delete ctx;
  return AEGIS_OK;
}

const char* aegis_last_error(const aegis_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }
void* aegis_stream_compute(aegis_ctx* ctx) { return ctx ? (void*)ctx->c->stream : nullptr; }
void* aegis_stream_comm(aegis_ctx* ctx) { return ctx ? (void*)ctx->c->comm : nullptr; }
int aegis_sync(aegis_ctx* ctx) {
  return guard(ctx, [&] { AEGIS_CHECK_CUDA(cudaStreamSynchronize(ctx->c->stream)); });
}
uint64_t aegis_prime(const aegis_ctx* ctx, uint32_t e) { return e < aegis::kNumExt ? ctx->c->prime(e) : 0; }
uint64_t aegis_launch_count(const aegis_ctx* ctx) { return ctx ? ctx->c->launches : 0; }

int aegis_bundle_alloc(aegis_ctx* ctx, uint32_t lanes, uint32_t comps, uint32_t level, aegis_bundle** out) {
  return guard(ctx, [&] {
    if (!out || !lanes || !comps || comps > 3) throw Error(AEGIS_EINVAL, "bad bundle shape");
    if (level == 0) throw Error(AEGIS_EINVAL, "exhausted modulus chain");
    if (level > ctx->c->chain) throw Error(AEGIS_EINVAL, "ciphertext level exceeds chain_length");
    auto* h = new aegis_bundle;
    try {
      h->b = ctx->c->new_bundle(lanes, comps, level, true);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}
int aegis_bundle_free(aegis_ctx* ctx, aegis_bundle* b) {
  return guard(ctx, [&] {
    if (b) ctx->c->free_bundle(b->b);
    delete b;
  });
}
int aegis_bundle_upload(aegis_ctx* ctx, aegis_bundle* b, const uint64_t* host, uint64_t count) {
  return guard(ctx, [&] {
    Bundle& bb = need(b);
    if (count * 8 != bb.bytes) throw Error(AEGIS_EINVAL, "upload size mismatch");
    AEGIS_CHECK_CUDA(cudaMemcpyAsync(bb.ptr, host, bb.bytes, cudaMemcpyHostToDevice, ctx->c->stream));
  });
}
int aegis_bundle_download(aegis_ctx* ctx, const aegis_bundle* b, uint64_t* host, uint64_t count) {
  return guard(ctx, [&] {
    const Bundle& bb = need(b);
    if (count * 8 != bb.bytes) throw Error(AEGIS_EINVAL, "download size mismatch");
    AEGIS_CHECK_CUDA(cudaMemcpyAsync(host, bb.ptr, bb.bytes, cudaMemcpyDeviceToHost, ctx->c->stream));
    AEGIS_CHECK_CUDA(cudaStreamSynchronize(ctx->c->stream));
  });
}
int aegis_bundle_info(const aegis_bundle* b, uint32_t* lanes, uint32_t* comps, uint32_t* level, uint64_t* ptr) {
  if (!b || !b->b) return AEGIS_EINVAL;
  if (lanes) *lanes = b->b->lanes;
  if (comps) *comps = b->b->comps;
  if (level) *level = b->b->level;
  if (ptr) *ptr = (uint64_t)(uintptr_t)b->b->ptr;
  return AEGIS_OK;
}
int aegis_bundle_fill_input(aegis_ctx* ctx, aegis_bundle* b, uint32_t bundle_id) {
  return guard(ctx, [&] {
    Bundle& bb = need(b);
    Context& c = *ctx->c;
    AEGIS_CHECK_CUDA(aegis::launch_fill_uniform(bb.view(), bb.lanes, bb.comps, bb.level, c.n, c.seed_input, 1, bundle_id,
                                                c.d_ident, c.d_pc, c.stream));
    c.count();
  });
}
int aegis_bundle_hash(aegis_ctx* ctx, const aegis_bundle* b, uint32_t comps, uint32_t level, uint64_t* out) {
  return guard(ctx, [&] {
    const Bundle& bb = need(b);
    if (comps > bb.comps || level > bb.level) throw Error(AEGIS_EINVAL, "hash range exceeds bundle");
    Context& c = *ctx->c;
    u64* d = c.alloc(1);
    AEGIS_CHECK_CUDA(cudaMemsetAsync(d, 0, 8, c.stream));
    AEGIS_CHECK_CUDA(aegis::launch_hash(bb.view(), bb.lanes, comps, level, c.n, (unsigned long long*)d, c.stream));
    c.count();
    AEGIS_CHECK_CUDA(cudaMemcpyAsync(out, d, 8, cudaMemcpyDeviceToHost, c.stream));
    AEGIS_CHECK_CUDA(cudaStreamSynchronize(c.stream));
    c.release(d);
  });
}

int aegis_keys_generate(aegis_ctx* ctx, const uint64_t* ids, uint32_t count) {
  return guard(ctx, [&] {
    for (uint32_t i = 0; i < count; ++i) ctx->c->generate_key(ids[i]);
  });
}
int aegis_keys_bytes(const aegis_ctx* ctx, uint64_t* out) {
  if (!ctx || !out) return AEGIS_EINVAL;
  *out = ctx->c->total_key_bytes();
  return AEGIS_OK;
}

int aegis_ntt(aegis_ctx* ctx, aegis_bundle* b, uint32_t lane, uint32_t lane_count, uint32_t lo, uint32_t hi,
              int inverse) {
  return guard(ctx, [&] {
    Bundle& bb = need(b);
    check_lanes(bb, lane, lane_count, "ntt");
    if (lo > hi || hi >= bb.level) throw Error(AEGIS_EINVAL, "ntt: prime range out of bounds");
    std::vector<u32> off, pr;
    for (u32 cp = 0; cp < bb.comps; ++cp)
      for (u32 i = lo; i <= hi; ++i) {
        off.push_back(cp * bb.level + i);
        pr.push_back(i);
      }
    ctx->c->ntt(bb.view().limb(lane, 0, 0, ctx->c->n), (size_t)bb.comps * bb.level * ctx->c->n, lane_count, off, pr,
                inverse != 0);
  });
}

int aegis_automorphism(aegis_ctx* ctx, aegis_bundle* out, const aegis_bundle* in, uint32_t lane, uint32_t count,
                       uint32_t level, uint64_t galois) {
  return guard(ctx, [&] {
    Bundle& o = need(out);
    const Bundle& i = need(in);
    check_lanes(o, lane, count, "automorphism");
    check_lanes(i, lane, count, "automorphism");
    check_level(i, level, "automorphism");
    check_level(o, level, "automorphism");
    if (!(galois & 1)) throw Error(AEGIS_EINVAL, "galois element must be odd");
    const u32 nc = std::min(o.comps, i.comps);
    AEGIS_CHECK_CUDA(aegis::launch_automorphism(o.view(), LaneMap{lane, count}, i.view(), LaneMap{lane, count}, count,
                                                nc, level, ctx->c->log_n, galois, ctx->c->stream));
    ctx->c->count();
  });
}

int aegis_basis_convert(aegis_ctx* ctx, aegis_bundle* out, const aegis_bundle* in, const uint32_t* src_ext,
                        const uint32_t* src_limb, uint32_t k, const uint32_t* dst_ext, const uint32_t* dst_limb,
                        uint32_t m) {
  return guard(ctx, [&] {
    Bundle& o = need(out);
    const Bundle& i = need(in);
    if (o.lanes != i.lanes || o.comps != i.comps) throw Error(AEGIS_EINVAL, "basis_convert: shape mismatch");
    for (u32 t = 0; t < k; ++t)
      if (src_limb[t] >= i.level || src_ext[t] >= aegis::kNumExt) throw Error(AEGIS_EINVAL, "basis_convert: bad source");
    for (u32 t = 0; t < m; ++t)
      if (dst_limb[t] >= o.level || dst_ext[t] >= aegis::kNumExt) throw Error(AEGIS_EINVAL, "basis_convert: bad target");
    const u32 n = ctx->c->n;
    for (u32 cp = 0; cp < i.comps; ++cp)
      ctx->c->basis_convert(i.view().limb(0, cp, 0, n), (size_t)i.comps * i.level * n,
                            std::vector<u32>(src_limb, src_limb + k), std::vector<u32>(src_ext, src_ext + k),
                            o.view().limb(0, cp, 0, n), (size_t)o.comps * o.level * n,
                            std::vector<u32>(dst_limb, dst_limb + m), std::vector<u32>(dst_ext, dst_ext + m), i.lanes);
  });
}

int aegis_keyswitch(aegis_ctx* ctx, aegis_bundle* out, const aegis_bundle* in, uint32_t comp, uint32_t level,
                    uint64_t key_id) {
  return guard(ctx, [&] {
    Bundle& o = need(out);
    const Bundle& i = need(in);
    if (comp >= i.comps || o.comps < 2 || o.lanes != i.lanes) throw Error(AEGIS_EINVAL, "keyswitch: bad shapes");
    check_level(i, level, "keyswitch");
    check_level(o, level, "keyswitch");
    const u32 n = ctx->c->n;
    Context::KsOut ko;
    ko.out[0] = o.view().limb(0, 0, 0, n);
    ko.out[1] = o.view().limb(0, 1, 0, n);
    ko.out_lane[0] = ko.out_lane[1] = (size_t)o.comps * o.level * n;
    ko.add[0] = ko.add[1] = nullptr;
    ko.add_lane[0] = ko.add_lane[1] = 0;
    Context& c = *ctx->c;
    if (key_id >= 500) {
      // rotation keys are stored as key' = auto_{k^-1}(key): KS(d, key) = auto_k(KS(auto_{k^-1}(d), key'))
      const u64 gk = c.galois_of((int)((long long)key_id - 1000));
      u64 ginv = 1, b = gk, e = c.n - 1;
      while (e) {
        if (e & 1) ginv = (ginv * b) % (2ull * c.n);
        b = (b * b) % (2ull * c.n);
        e >>= 1;
      }
      u64* tmp2 = c.alloc((size_t)i.lanes * level * n);
      // component `comp` of every lane: a view based at that component keeps the lane stride
      aegis::View sv{i.view().limb(0, comp, 0, n), i.lanes, i.comps, i.level};
      AEGIS_CHECK_CUDA(aegis::launch_automorphism(aegis::View{tmp2, i.lanes, 1, level}, LaneMap{0, i.lanes}, sv,
                                                  LaneMap{0, i.lanes}, i.lanes, 1, level, c.log_n, ginv, c.stream));
      c.count();
      c.keyswitch(tmp2, (size_t)level * n, i.lanes, level, key_id, ko, gk);
      c.release(tmp2);
      return;
    }
    c.keyswitch(i.view().limb(0, comp, 0, n), (size_t)i.comps * i.level * n, i.lanes, level, key_id, ko);
  });
}

int aegis_rot(aegis_ctx* ctx, aegis_bundle* out, uint32_t out_lane, const aegis_bundle* in, uint32_t in_lane,
              uint32_t lanes, uint32_t level, int offset) {
  return guard(ctx, [&] {
    Bundle& o = need(out);
    const Bundle& i = need(in);
    check_lanes(o, out_lane, lanes, "rot");
    check_lanes(i, in_lane, lanes, "rot");
    check_level(i, level, "rot");
    check_level(o, level, "rot");
    ctx->c->op_rot(o, out_lane, i, LaneMap{in_lane, lanes}, lanes, level, offset);
  });
}
int aegis_relin(aegis_ctx* ctx, aegis_bundle* b, uint32_t lane, uint32_t lanes, uint32_t level) {
  return guard(ctx, [&] {
    Bundle& bb = need(b);
    check_lanes(bb, lane, lanes, "relin");
    check_level(bb, level, "relin");
    ctx->c->op_relin(bb, lane, lanes, level);
  });
}
int aegis_rescale(aegis_ctx* ctx, aegis_bundle* out, uint32_t out_lane, const aegis_bundle* in, uint32_t in_lane,
                  uint32_t lanes, uint32_t level) {
  return guard(ctx, [&] {
    Bundle& o = need(out);
    const Bundle& i = need(in);
    check_lanes(o, out_lane, lanes, "rescale");
    check_lanes(i, in_lane, lanes, "rescale");
    check_level(i, level, "rescale");
    if (level < 2) throw Error(AEGIS_EINVAL, "level underflow: cannot rescale below level 1");
    check_level(o, level - 1, "rescale");
    ctx->c->op_rescale(o, out_lane, i, LaneMap{in_lane, lanes}, lanes, level);
  });
}
int aegis_boot(aegis_ctx* ctx, aegis_bundle* out, uint32_t out_lane, const aegis_bundle* in, uint32_t in_lane,
               uint32_t lanes, uint32_t level, uint32_t out_level) {
  return guard(ctx, [&] {
    Bundle& o = need(out);
    const Bundle& i = need(in);
    check_lanes(o, out_lane, lanes, "boot");
    check_lanes(i, in_lane, lanes, "boot");
    check_level(i, level, "boot");
    check_level(o, out_level, "boot");
    ctx->c->op_boot(o, out_lane, i, LaneMap{in_lane, lanes}, lanes, level, out_level);
  });
}
int aegis_cmult(aegis_ctx* ctx, aegis_bundle* out, uint32_t out_lane, uint32_t lanes, const aegis_bundle* a,
                uint32_t a_lane, uint32_t a_count, const aegis_bundle* b, uint32_t b_lane, uint32_t b_count,
                uint32_t level) {
  return guard(ctx, [&] {
    Bundle& o = need(out);
    const Bundle& A = need(a);
    const Bundle& Bb = need(b);
    check_lanes(o, out_lane, lanes, "cmult");
    check_lanes(A, a_lane, a_count, "cmult");
    check_lanes(Bb, b_lane, b_count, "cmult");
    if (!a_count || !b_count) throw Error(AEGIS_EINVAL, "cmult: empty operand");
    check_level(A, level, "cmult");
    check_level(Bb, level, "cmult");
    check_level(o, level, "cmult");
    ctx->c->op_cmult(o, out_lane, lanes, A, LaneMap{a_lane, a_count}, Bb, LaneMap{b_lane, b_count}, level);
  });
}
int aegis_cadd(aegis_ctx* ctx, aegis_bundle* out, uint32_t out_lane, uint32_t lanes, const aegis_bundle* a,
               uint32_t a_lane, uint32_t a_count, const aegis_bundle* b, uint32_t b_lane, uint32_t b_count,
               uint32_t level, int accumulate) {
  return guard(ctx, [&] {
    Bundle& o = need(out);
    const Bundle& A = need(a);
    check_lanes(o, out_lane, lanes, "cadd");
    check_lanes(A, a_lane, a_count, "cadd");
    check_level(A, level, "cadd");
    check_level(o, level, "cadd");
    const Bundle* Bp = nullptr;
    if (!accumulate) {
      Bp = &need(b);
      check_lanes(*Bp, b_lane, b_count, "cadd");
      check_level(*Bp, level, "cadd");
    }
    if (!a_count || (!accumulate && !b_count)) throw Error(AEGIS_EINVAL, "cadd: empty operand");
    ctx->c->op_cadd(o, out_lane, lanes, A, LaneMap{a_lane, a_count}, Bp, LaneMap{b_lane, b_count ? b_count : 1}, level,
                    accumulate != 0);
  });
}
int aegis_pmult_acc(aegis_ctx* ctx, aegis_bundle* acc, uint32_t acc_lane, uint32_t acc_lanes, uint32_t chunk_period,
                    const aegis_bundle* x, uint32_t x_lane, uint32_t x_lanes, uint32_t wb, uint32_t wlanes,
                    uint32_t level) {
  return guard(ctx, [&] {
    Bundle& A = need(acc);
    const Bundle& X = need(x);
    check_lanes(A, acc_lane, acc_lanes, "pmult");
    check_lanes(X, x_lane, x_lanes, "pmult");
    check_level(A, level, "pmult");
    check_level(X, level, "pmult");
    ctx->c->op_pmult(A, acc_lane, acc_lanes, chunk_period, X, x_lane, x_lanes, wb, wlanes, level);
  });
}

// ---- graphs ----------------------------------------------------------------
namespace {
void build_graph(const aegis_params& p, const aegis_model* m, aegis_graph** out) {
  if (!m || !out) throw Error(AEGIS_EINVAL, "null argument");
  if (p.log_n < 4 || p.log_n > AEGIS_MAX_LOG_N) throw Error(AEGIS_EINVAL, "ring_degree must be a power of two");
  if (p.chain_length == 0) throw Error(AEGIS_EINVAL, "chain_length must be positive");
  if (p.bootstrap_level > p.chain_length) throw Error(AEGIS_EINVAL, "bootstrap_level exceeds chain_length");
  struct { u32 n, chain, lboot; } c{1u << p.log_n, p.chain_length, p.bootstrap_level};
  {
    hp::CkksProfile prof;
    prof.ring_degree = c.n;
    prof.slot_count = c.n / 2;
    prof.chain_length = c.chain;
    prof.special_prime_count = aegis::kAlpha;
    prof.bootstrap_level = c.lboot;
    hp::PackingLayout lay{m->slots_per_token, m->model_dim, m->head_dim};
    if (!lay.slots_per_token || !lay.model_dim || !lay.head_dim)
      throw Error(AEGIS_EINVAL, "layout dimensions must be positive");
    if (lay.slots_per_token > prof.slot_count || prof.slot_count % lay.slots_per_token)
      throw Error(AEGIS_EINVAL, "slot_count must be divisible by slots_per_token (full slot utilization)");
    hp::TransformerConfig cfg;
    cfg.layer_count = m->layers;
    cfg.model_dim = m->model_dim;
    cfg.ffn_dim = m->ffn_dim;
    hp::AppGraph app = m->kind == 1 ? hp::build_ffn_graph(cfg, prof, m->tokens)
                                    : hp::build_transformer_graph(cfg, prof, m->tokens);
    auto* g = new aegis_graph;
    g->g = hp::lower_app_to_he(app, prof, lay);
    std::ostringstream h;
    h << "# heops v1 N=" << c.n << " L=" << c.chain << " K=" << aegis::kAlpha << " lboot=" << c.lboot
      << " stok=" << m->slots_per_token << " d=" << m->model_dim << " hd=" << m->head_dim << " dff=" << m->ffn_dim
      << " T=" << m->tokens << " layers=" << m->layers << " kind=" << m->kind << " exact=0";
    g->header = h.str();
    *out = g;
  }
}
}  // namespace

int aegis_graph_build(aegis_ctx* ctx, const aegis_model* m, aegis_graph** out) {
  return guard(ctx, [&] {
    aegis_params p{ctx->c->log_n, ctx->c->chain, aegis::kAlpha, ctx->c->lboot, 0, 0, 0};
    build_graph(p, m, out);
  });
}
int aegis_graph_build_params(const aegis_params* p, const aegis_model* m, aegis_graph** out) {
  if (!p) return AEGIS_EINVAL;
  return guard(nullptr, [&] { build_graph(*p, m, out); });
}
int aegis_graph_load(aegis_ctx* ctx, const char* path, aegis_graph** out) {
  return guard(ctx, [&] {
    std::ifstream f(path);
    if (!f) throw Error(AEGIS_EINVAL, std::string("cannot open ") + path);
    std::stringstream ss;
    ss << f.rdbuf();
    auto* g = new aegis_graph;
    try {
      g->g = hp::parse_heops(ss.str());
    } catch (...) {
      delete g;
      throw;
    }
    const std::string s = ss.str();
    g->header = s.substr(0, s.find('\n'));
    *out = g;
  });
}
int aegis_graph_dump(const aegis_graph* g, const char* path) {
  if (!g || !path) return AEGIS_EINVAL;
  std::ofstream f(path);
  if (!f) return AEGIS_EINVAL;
  f << hp::dump_heops(g->g, g->header);
  return f ? AEGIS_OK : AEGIS_EINVAL;
}
int aegis_graph_info(const aegis_graph* g, uint64_t* ops, uint64_t* bundles) {
  if (!g) return AEGIS_EINVAL;
  if (ops) *ops = g->g.ops.size();
  if (bundles) *bundles = g->g.bundles.size();
  return AEGIS_OK;
}
int aegis_graph_set_shard(aegis_graph* g, uint32_t lo, uint32_t hi) {
  if (!g || lo >= hi) return AEGIS_EINVAL;
  g->shard_lo = lo;
  g->shard_hi = hi;
  return AEGIS_OK;
}
int aegis_graph_key_ids(const aegis_graph* g, uint64_t* ids, uint32_t cap, uint32_t* n) {
  if (!g || !n) return AEGIS_EINVAL;
  std::set<uint64_t> s;
  for (const hp::HeOp& op : g->g.ops) {
    if (op.kind == hp::HeOpKind::kRot) s.insert(1000u + (uint64_t)(int64_t)op.rot_offset);
    if (op.kind == hp::HeOpKind::kRelin) s.insert(0);
  }
  uint32_t k = 0;
  for (uint64_t v : s) {
    if (ids && k < cap) ids[k] = v;
    ++k;
  }
  *n = k;
  return AEGIS_OK;
}
int aegis_graph_run(aegis_ctx* ctx, aegis_graph* g, int64_t max_ops, uint64_t* hashes, uint64_t nhashes) {
  return guard(ctx, [&] {
    if (!g) throw Error(AEGIS_EINVAL, "null graph");
    Context& c = *ctx->c;
    const size_t nb = g->g.bundles.size();
    Exec ex(c, g->g);
    c.peak_bytes = c.live_bytes;
    u64* dh = nullptr;
    if (hashes) {
      dh = c.alloc(nb);
      AEGIS_CHECK_CUDA(cudaMemsetAsync(dh, 0, nb * 8, c.stream));
      ex.d_hash = (unsigned long long*)dh;
    }
    ex.run(max_ops);
    if (hashes) {
      std::vector<u64> h(nb);
      AEGIS_CHECK_CUDA(cudaMemcpyAsync(h.data(), dh, nb * 8, cudaMemcpyDeviceToHost, c.stream));
      AEGIS_CHECK_CUDA(cudaStreamSynchronize(c.stream));
      for (size_t i = 0; i < nb && i < nhashes; ++i) hashes[i] = h[i];
      c.release(dh);
    }
    g->peak = c.peak_bytes;
  });
}
int aegis_graph_io_words(const aegis_graph* g, uint64_t* in_words, uint64_t* out_words) {
  if (!g) return AEGIS_EINVAL;
  // N is not stored in the graph: infer from the header ("N=<n>")
  const size_t pos = g->header.find(" N=");
  const uint64_t n = pos == std::string::npos ? 0 : std::stoull(g->header.substr(pos + 3));
  uint64_t win = 0;
  for (u32 b : g->g.graph_inputs) win += (uint64_t)g->g.bundles[b].lanes * 2 * g->g.bundles[b].level * n;
  uint64_t wout = 0;
  if (!g->g.ops.empty()) {
    const hp::CtBundle& fb = g->g.bundles[g->g.ops.back().out.bundle];
    wout = (uint64_t)fb.lanes * 2 * fb.level * n;
  }
  if (in_words) *in_words = win;
  if (out_words) *out_words = wout;
  return AEGIS_OK;
}
int aegis_graph_host_inputs(aegis_ctx* ctx, const aegis_graph* g, uint64_t* in, uint64_t in_words) {
  return guard(ctx, [&] {
    if (!g || !in) throw Error(AEGIS_EINVAL, "null argument");
    Context& c = *ctx->c;
    uint64_t need = 0;
    aegis_graph_io_words(g, &need, nullptr);
    if (need != in_words) throw Error(AEGIS_EINVAL, "host input size mismatch");
    size_t off = 0;
    for (u32 id : g->g.graph_inputs) {
      const hp::CtBundle& cb = g->g.bundles[id];
      for (u32 ln = 0; ln < cb.lanes; ++ln)
        for (u32 cp = 0; cp < 2; ++cp)
          for (u32 lb = 0; lb < cb.level; ++lb) {
            const u64 rk = aegis::row_key(c.seed_input, 1, id, ln, cp, lb);
            const u64 p = c.prime(lb);
            const u32 sh = (u32)__builtin_clzll(p);
            for (u32 x = 0; x < c.n; ++x) in[off++] = aegis::uniform_at(rk, x, p, sh);
          }
    }
  });
}
int aegis_graph_run_host(aegis_ctx* ctx, aegis_graph* g, const uint64_t* in, uint64_t in_words, uint64_t* out,
                         uint64_t out_words) {
  return guard(ctx, [&] {
    if (!g || !in || !out) throw Error(AEGIS_EINVAL, "null argument");
    uint64_t wi = 0, wo = 0;
    aegis_graph_io_words(g, &wi, &wo);
    if (wi != in_words || wo != out_words) throw Error(AEGIS_EINVAL, "host buffer size mismatch");
    Context& c = *ctx->c;
    Exec ex(c, g->g);
    c.peak_bytes = c.live_bytes;
    ex.host_in = reinterpret_cast<const u64*>(in);
    ex.host_out = reinterpret_cast<u64*>(out);
    ex.run(-1);
    AEGIS_CHECK_CUDA(cudaStreamSynchronize(c.stream));
    g->peak = c.peak_bytes;
  });
}
int aegis_graph_free(aegis_graph* g) {
  delete g;
  return AEGIS_OK;
}
uint64_t aegis_graph_peak_bytes(const aegis_graph* g) { return g ? g->peak : 0; }

}  // extern "C"

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
#include "executor.h"
#include "p2p.h"
#include "plan.h"
#include "heplan_ir.h"
#include "store.h"

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
struct aegis_p2p {
  std::unique_ptr<aegis::P2pWindow> w;
};

namespace {

thread_local std::string g_create_err;

// context-free calls (ctx == NULL) report through aegis_last_error(NULL)
template <class F>
int guard(aegis_ctx* ctx, F&& f) {
  std::string& err = ctx ? ctx->err : g_create_err;
  try {
    f();
    return AEGIS_OK;
  } catch (const Error& e) {
    err = e.what();
    return e.code;
  } catch (const std::invalid_argument& e) {
    err = e.what();
    return AEGIS_EINVAL;
  } catch (const std::logic_error& e) {
    err = e.what();
    return AEGIS_ELOGIC;
  } catch (const std::bad_alloc& e) {
    err = "host allocation failed";
    return AEGIS_EOOM;
  } catch (const std::exception& e) {
    err = e.what();
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
  std::unique_ptr<aegis::ShardPlan> shard;
  std::unique_ptr<aegis::ShardPlan> hash_lanes;  // aegis_graph_set_hash_group
  aegis::ReduceFn reduce = nullptr;
  aegis::P2pWindow* p2p = nullptr;  // device-synchronised exchange window (not owned)
  int fault = 0;
  int stored_weights = 0;
  int reference_modes = 0;
  void* reduce_user = nullptr;
  int hoist = 1;
  int dce = 0;
  int wrap_defer = 1;
  uint64_t h2d = 0, d2h = 0, comm = 0;
  bool profile = false;
  std::vector<float> op_ms;
  std::vector<float> comm_trace;
};

namespace {
// "# heops v1 N=65536 ... T=2048 ..." -> value of `key=`
uint64_t header_value(const std::string& h, const std::string& key) {
  const size_t pos = h.find(" " + key + "=");
  if (pos == std::string::npos) throw Error(AEGIS_EINVAL, "graph header lacks " + key);
  return std::stoull(h.substr(pos + key.size() + 2));
}
uint32_t token_groups(const aegis_graph* g) {
  const uint64_t n = header_value(g->header, "N"), T = header_value(g->header, "T"),
                 stok = header_value(g->header, "stok");
  const uint64_t per = n / 2 / stok;
  return (uint32_t)((T + per - 1) / per);
}
void run_graph(aegis_ctx* ctx, aegis_graph* g, aegis::RunOptions opt) {
  Context& c = *ctx->c;
  opt.shard = g->shard.get();
  opt.hash_lanes = g->hash_lanes.get();
  opt.reduce = g->reduce;
  opt.reduce_user = g->reduce_user;
  opt.p2p = g->shard && g->shard->m > 1 ? g->p2p : nullptr;
  opt.fault = g->fault;
  opt.stored_weights = g->stored_weights != 0;
  opt.reference_modes = g->reference_modes != 0;
  opt.hoist = g->hoist != 0;
  opt.dce = g->dce != 0;
  opt.wrap_defer = g->wrap_defer != 0;
  if (g->profile) {
    opt.op_ms = &g->op_ms;
    opt.comm_trace = &g->comm_trace;
  }
  // no trim here: the arena keeps its mapping across runs (re-mapping ~130 GB
  // per layer run stalled the stream); key allocation trims on demand
  c.peak_bytes = c.live_bytes;
  aegis::Executor ex(c, g->g, opt);
  ex.run();
  g->h2d = ex.h2d_bytes;
  g->comm = ex.comm_bytes;
  g->d2h = ex.d2h_bytes;
  g->peak = c.peak_bytes;
}
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

namespace {
aegis::KernelProbe g_probe_state;
}
int aegis_probe_start(aegis_ctx* ctx, int kind) {
  return guard(ctx, [&] {
    if (kind < 0 || kind > aegis::kProbeFwdBKm) throw Error(AEGIS_EINVAL, "unknown probe kind");
    AEGIS_CHECK_CUDA(cudaStreamSynchronize(ctx->c->stream));
    for (cudaEvent_t e : g_probe_state.ev) cudaEventDestroy(e);
    g_probe_state = aegis::KernelProbe{};
    g_probe_state.kind = kind;
    aegis::g_probe = kind ? &g_probe_state : nullptr;
  });
}
int aegis_probe_read(aegis_ctx* ctx, uint64_t* launches, double* ms, double* alg_bytes) {
  return guard(ctx, [&] {
    AEGIS_CHECK_CUDA(cudaStreamSynchronize(ctx->c->stream));
    double t = 0;
    for (size_t i = 0; i + 1 < g_probe_state.ev.size(); i += 2) {
      float x = 0;
      AEGIS_CHECK_CUDA(cudaEventElapsedTime(&x, g_probe_state.ev[i], g_probe_state.ev[i + 1]));
      t += x;
    }
    if (launches) *launches = g_probe_state.launches;
    if (ms) *ms = t;
    if (alg_bytes) *alg_bytes = g_probe_state.alg_bytes;
  });
}
int aegis_ntt_impl(int impl) {
  if (impl == aegis::kNttInt || impl == aegis::kNttF64) {
    aegis::g_ntt_impl = impl;
    aegis::g_ntt_v2 = 1;
  } else if (impl == 2) {  // FP64 butterflies through the generic (v1) passes
    aegis::g_ntt_impl = aegis::kNttF64;
    aegis::g_ntt_v2 = 0;
  }
  return aegis::g_ntt_impl == aegis::kNttF64 && !aegis::g_ntt_v2 ? 2 : aegis::g_ntt_impl;
}

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
    AEGIS_CHECK_CUDA(aegis::launch_hash(bb.view(), 0, bb.lanes, comps, level, c.n, (unsigned long long*)d, c.stream));
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
int aegis_keys_upload(aegis_ctx* ctx, uint64_t key_id, const uint64_t* host, uint64_t words, int coeff_domain) {
  return guard(ctx, [&] {
    if (!host) throw Error(AEGIS_EINVAL, "key upload: null host buffer");
    ctx->c->upload_key(key_id, reinterpret_cast<const aegis::u64*>(host), words, coeff_domain != 0);
  });
}
int aegis_bundle_save(aegis_ctx* ctx, const aegis_bundle* b, const char* path) {
  return guard(ctx, [&] {
    if (!path) throw Error(AEGIS_EINVAL, "null path");
    aegis::store_save_bundle(*ctx->c, need(b), path);
  });
}
int aegis_bundle_load(aegis_ctx* ctx, const char* path, aegis_bundle** out) {
  return guard(ctx, [&] {
    if (!path || !out) throw Error(AEGIS_EINVAL, "null argument");
    auto* h = new aegis_bundle;
    try {
      h->b = aegis::store_load_bundle(*ctx->c, path);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}
int aegis_keys_save(aegis_ctx* ctx, uint64_t key_id, const char* path) {
  return guard(ctx, [&] {
    if (!path) throw Error(AEGIS_EINVAL, "null path");
    aegis::store_save_key(*ctx->c, key_id, path);
  });
}
int aegis_keys_load(aegis_ctx* ctx, uint64_t key_id, const char* path) {
  return guard(ctx, [&] {
    if (!path) throw Error(AEGIS_EINVAL, "null path");
    aegis::store_load_key(*ctx->c, key_id, path);
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
    if (&o == &i) throw Error(AEGIS_EINVAL, "keyswitch: out must not alias in (the finish scatters over its input)");
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
    if (&o == &i && out_lane < in_lane + lanes && in_lane < out_lane + lanes)
      throw Error(AEGIS_EINVAL, "rot: output lanes overlap the input lanes (the automorphism scatter is not in-place)");
    ctx->c->op_rot(o, out_lane, i, LaneMap{in_lane, lanes}, lanes, level, offset);
  });
}
int aegis_rot_hoisted(aegis_ctx* ctx, aegis_bundle* const* outs, const uint32_t* out_lanes, const int* offsets,
                      uint32_t n_off, const aegis_bundle* in, uint32_t in_lane, uint32_t lanes, uint32_t level) {
  return guard(ctx, [&] {
    const Bundle& i = need(in);
    if (!n_off) return;
    if (!outs || !out_lanes || !offsets) throw Error(AEGIS_EINVAL, "rot_hoisted: null argument");
    check_lanes(i, in_lane, lanes, "rot_hoisted");
    check_level(i, level, "rot_hoisted");
    if (i.comps < 2) throw Error(AEGIS_EINVAL, "rot_hoisted: the source must be a ciphertext");
    for (u32 k = 0; k < n_off; ++k) {
      Bundle& o = need(outs[k]);
      check_lanes(o, out_lanes[k], lanes, "rot_hoisted");
      check_level(o, level, "rot_hoisted");
      if (o.comps < 2) throw Error(AEGIS_EINVAL, "rot_hoisted: outputs must have 2 components");
      if (&o == &i && out_lanes[k] < in_lane + lanes && in_lane < out_lanes[k] + lanes)
        throw Error(AEGIS_EINVAL, "rot_hoisted: output lanes overlap the input lanes");
      Context::rotation_key_id(offsets[k]);  // offset range check before any work
    }
    Context& c = *ctx->c;
    // ModUp(c1) once per lane batch, shared by every offset (bit-identical to
    // the per-rotation ModUp: the key is pre-permuted)
    const size_t per_lane = c.modup_words_per_lane(level);
    const u32 batch = (u32)std::max<size_t>(1, std::min<size_t>(lanes, c.ws_budget(2) / (per_lane * 8)));
    u64* ext = c.alloc(per_lane * batch);
    try {
      const size_t in_ls = (size_t)i.comps * i.level * c.n;
      for (u32 done = 0; done < lanes; done += batch) {
        const u32 cnt = std::min(batch, lanes - done);
        c.modup(i.view().limb(in_lane + done, 1, 0, c.n), in_ls, cnt, level, ext);
        for (u32 k = 0; k < n_off; ++k)
          c.op_rot_cached(*outs[k]->b, out_lanes[k] + done, i, LaneMap{in_lane + done, cnt}, cnt, level,
                          offsets[k], ext);
      }
    } catch (...) {
      c.release(ext);
      throw;
    }
    c.release(ext);
  });
}
int aegis_padd(aegis_ctx* ctx, aegis_bundle* out, uint32_t out_lane, uint32_t lanes, const aegis_bundle* ct,
               uint32_t ct_lane, uint32_t ct_count, const aegis_bundle* pt, uint32_t pt_lane, uint32_t pt_count,
               uint32_t level) {
  return guard(ctx, [&] {
    const Bundle& P = need(pt);
    const Bundle& C = need(ct);
    if (P.comps != 1) throw Error(AEGIS_EINVAL, "padd: the plaintext operand must have 1 component");
    if (C.comps < 2) throw Error(AEGIS_EINVAL, "padd: the ciphertext operand must have 2 components");
    if (level == 0) throw Error(AEGIS_EINVAL, "exhausted modulus chain");
    const int rc = aegis_limb_op(ctx, AEGIS_LIMB_ADD, out, out_lane, lanes, ct, ct_lane, ct_count, pt, pt_lane,
                                 pt_count, 0, level - 1, 0);
    if (rc) throw Error(rc, ctx->err);
  });
}
int aegis_encode(aegis_ctx* ctx, aegis_bundle* pt, uint32_t lane, uint32_t lanes, uint32_t level, uint32_t wb) {
  return guard(ctx, [&] {
    Bundle& P = need(pt);
    check_lanes(P, lane, lanes, "encode");
    check_level(P, level, "encode");
    if (P.comps != 1) throw Error(AEGIS_EINVAL, "encode: plaintext bundles have 1 component");
    Context& c = *ctx->c;
    AEGIS_CHECK_CUDA(aegis::launch_limb_generate(P.view(), lane, lanes, 1, 0, level, c.n, c.seed_weight, 2, wb, c.d_pc,
                                                 c.stream));
    c.count();
  });
}
int aegis_limb_op(aegis_ctx* ctx, int opcode, aegis_bundle* out, uint32_t out_lane, uint32_t lanes,
                  const aegis_bundle* a, uint32_t a_lane, uint32_t a_count, const aegis_bundle* b, uint32_t b_lane,
                  uint32_t b_count, uint32_t lo, uint32_t hi, uint64_t param) {
  return guard(ctx, [&] {
    Bundle& o = need(out);
    Context& c = *ctx->c;
    check_lanes(o, out_lane, lanes, "limb_op");
    if (lo > hi || hi >= o.level) throw Error(AEGIS_EINVAL, "limb_op: prime range outside the output's limbs");
    const u32 limbs = hi - lo + 1;
    if (opcode == AEGIS_LIMB_KEYMUL)
      throw Error(AEGIS_EINVAL, "limb_op: kKeyMul runs inside aegis_keyswitch (the IR's KeyMul has no digit split)");
    if (opcode == AEGIS_LIMB_GENERATE) {
      AEGIS_CHECK_CUDA(aegis::launch_limb_generate(o.view(), out_lane, lanes, o.comps, lo, limbs, c.n, c.seed_weight,
                                                   2, param, c.d_pc, c.stream));
      c.count();
      return;
    }
    if (opcode < AEGIS_LIMB_ADD || opcode > AEGIS_LIMB_ADDACC) throw Error(AEGIS_EINVAL, "limb_op: unknown opcode");
    const Bundle& A = need(a);
    check_lanes(A, a_lane, a_count, "limb_op");
    if (!a_count) throw Error(AEGIS_EINVAL, "limb_op: empty operand");
    if (hi >= A.level) throw Error(AEGIS_EINVAL, "limb_op: prime range outside an operand's limbs");
    const bool two = opcode != AEGIS_LIMB_ADDACC;
    const Bundle* B = nullptr;
    if (two) {
      B = &need(b);
      check_lanes(*B, b_lane, b_count, "limb_op");
      if (!b_count) throw Error(AEGIS_EINVAL, "limb_op: empty operand");
      if (hi >= B->level) throw Error(AEGIS_EINVAL, "limb_op: prime range outside an operand's limbs");
    }
    const u32 ac = std::min<u32>(A.comps, 2), bc = B ? std::min<u32>(B->comps, 2) : 0;
    if (A.comps > 2 || (B && B->comps > 2)) throw Error(AEGIS_EINVAL, "limb_op: operands have at most 2 components");
    const bool mul = opcode == AEGIS_LIMB_MUL || opcode == AEGIS_LIMB_MULACC;
    const u32 oc = opcode == AEGIS_LIMB_ADDACC ? o.comps : (mul && ac == 2 && bc == 2 ? 3 : std::max(ac, bc));
    if (oc > o.comps) throw Error(AEGIS_EINVAL, "limb_op: the output has too few components");
    auto overlaps = [&](const Bundle& X, u32 xl, u32 xc) {
      return &X == &o && xl < out_lane + lanes && out_lane < xl + xc && !(xl == out_lane && xc == lanes);
    };
    if (overlaps(A, a_lane, a_count) || (B && overlaps(*B, b_lane, b_count)))
      throw Error(AEGIS_EINVAL, "limb_op: the output overlaps an operand with different lanes");
    const aegis::View bv = B ? B->view() : A.view();
    AEGIS_CHECK_CUDA(aegis::launch_limb_op(opcode, o.view(), out_lane, oc, A.view(), LaneMap{a_lane, a_count}, ac, bv,
                                           LaneMap{b_lane, b_count ? b_count : 1}, bc, lanes, lo, limbs, c.n, c.d_pc,
                                           c.stream));
    c.count();
  });
}
int aegis_limb_drop(aegis_ctx* ctx, aegis_bundle* out, uint32_t out_lane, const aegis_bundle* in, uint32_t in_lane,
                    uint32_t lanes, uint32_t level, int mode) {
  if (mode == AEGIS_MODE_RESCALE_TAIL) return aegis_rescale(ctx, out, out_lane, in, in_lane, lanes, level);
  return guard(ctx, [&] {
    if (mode != AEGIS_MODE_NONE) throw Error(AEGIS_EINVAL, "limb_drop: mode must be kNone or kRescaleTail");
    Bundle& o = need(out);
    const Bundle& i = need(in);
    check_lanes(o, out_lane, lanes, "limb_drop");
    check_lanes(i, in_lane, lanes, "limb_drop");
    check_level(i, level, "limb_drop");
    if (level < 2) throw Error(AEGIS_EINVAL, "level underflow: cannot drop below level 1");
    check_level(o, level - 1, "limb_drop");
    if (o.comps < i.comps) throw Error(AEGIS_EINVAL, "limb_drop: the output has too few components");
    if (&o == &i && in_lane == out_lane) return;  // the dropped limb is simply no longer read
    if (&o == &i && out_lane < in_lane + lanes && in_lane < out_lane + lanes)
      throw Error(AEGIS_EINVAL, "limb_drop: output lanes overlap the input lanes");
    Context& c = *ctx->c;
    AEGIS_CHECK_CUDA(aegis::launch_copy(o.view(), out_lane, i.view(), LaneMap{in_lane, lanes}, lanes, i.comps,
                                        level - 1, 0, c.n, c.stream));
    c.count();
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
namespace {
std::string header_of(const aegis_graph_meta& m) {
  std::ostringstream h;
  h << "# heops v1 N=" << (1u << m.log_n) << " L=" << m.chain_length << " K=" << aegis::kAlpha
    << " lboot=" << m.bootstrap_level << " stok=" << m.slots_per_token << " d=" << m.model_dim
    << " hd=" << m.head_dim << " dff=" << m.ffn_dim << " T=" << m.tokens << " layers=" << m.layers
    << " kind=" << m.kind << " exact=0";
  return h.str();
}
}  // namespace
int aegis_graph_from_ops(const aegis_graph_meta* meta, const aegis_bundle_desc* bundles, uint32_t nb,
                         const aegis_op_desc* ops, uint64_t nops, const uint32_t* inputs, uint32_t ninputs,
                         aegis_graph** out) {
  return guard(nullptr, [&] {
    if (!meta || !out || (nb && !bundles) || (nops && !ops) || (ninputs && !inputs))
      throw Error(AEGIS_EINVAL, "graph_from_ops: null argument");
    if (meta->log_n < 4 || meta->log_n > AEGIS_MAX_LOG_N) throw Error(AEGIS_EINVAL, "ring_degree must be a power of two");
    if (!meta->slots_per_token) throw Error(AEGIS_EINVAL, "layout dimensions must be positive");
    auto g = std::make_unique<aegis_graph>();
    g->g.bundles.reserve(nb);
    for (uint32_t i = 0; i < nb; ++i) {
      const aegis_bundle_desc& d = bundles[i];
      hp::CtBundle b;
      b.id = i;
      b.lanes = d.lanes;
      b.level = d.level;
      b.components = d.components;
      if (d.cls > (uint32_t)hp::BundleClass::kScore || d.aggregation > (uint32_t)hp::AggregationAxis::kHeadWise)
        throw Error(AEGIS_EINVAL, "graph_from_ops: bundle " + std::to_string(i) + " has an unknown class");
      b.cls = (hp::BundleClass)d.cls;
      b.aggregation = (hp::AggregationAxis)d.aggregation;
      b.app_node = d.app_node;
      b.chunk_period = d.chunk_period;
      b.replicate_hint = d.replicate_hint != 0;
      if (d.tag) b.tag = d.tag;
      g->g.bundles.push_back(std::move(b));
    }
    g->g.ops.reserve(nops);
    for (uint64_t i = 0; i < nops; ++i) {
      const aegis_op_desc& d = ops[i];
      if (d.in_count > AEGIS_MAX_OP_INPUTS) throw Error(AEGIS_EINVAL, "heops: op " + std::to_string(i) + ": too many operands");
      if (d.kind > (uint32_t)hp::HeOpKind::kBoot) throw Error(AEGIS_EINVAL, "heops: op " + std::to_string(i) + ": unknown kind");
      hp::HeOp op;
      op.id = (uint32_t)i;
      op.kind = (hp::HeOpKind)d.kind;
      op.rot_offset = d.rot_offset;
      op.out = hp::LaneSlice{d.out.bundle, d.out.lane, d.out.lane_count};
      for (uint32_t k = 0; k < d.in_count; ++k) op.ins.push_back(hp::LaneSlice{d.ins[k].bundle, d.ins[k].lane, d.ins[k].lane_count});
      op.accumulate = d.accumulate != 0;
      op.aligned = d.aligned != 0;
      op.phase = d.phase;
      op.work = d.work;
      op.use_level = d.use_level;
      op.app_node = d.app_node;
      if (d.aggregation > (uint32_t)hp::AggregationAxis::kHeadWise)
        throw Error(AEGIS_EINVAL, "heops: op " + std::to_string(i) + ": unknown aggregation axis");
      op.aggregation = (hp::AggregationAxis)d.aggregation;
      g->g.ops.push_back(std::move(op));
    }
    g->g.graph_inputs.assign(inputs, inputs + ninputs);
    hp::validate_heops(g->g);
    g->header = header_of(*meta);
    *out = g.release();
  });
}
int aegis_graph_export(const aegis_graph* g, aegis_bundle_desc* bundles, uint32_t bcap, aegis_op_desc* ops,
                       uint64_t ocap, uint32_t* inputs, uint32_t icap, uint32_t* n_inputs, aegis_graph_meta* meta) {
  return guard(nullptr, [&] {
    if (!g) throw Error(AEGIS_EINVAL, "null graph");
    if ((bundles && bcap < g->g.bundles.size()) || (ops && ocap < g->g.ops.size()) ||
        (inputs && icap < g->g.graph_inputs.size()))
      throw Error(AEGIS_EINVAL, "graph_export: buffer too small");
    if (bundles)
      for (size_t i = 0; i < g->g.bundles.size(); ++i) {
        const hp::CtBundle& b = g->g.bundles[i];
        bundles[i] = aegis_bundle_desc{b.lanes, b.level, b.components, (uint32_t)b.cls, (uint32_t)b.aggregation,
                                       b.app_node, b.chunk_period, (uint32_t)b.replicate_hint, b.tag.c_str()};
      }
    if (ops)
      for (size_t i = 0; i < g->g.ops.size(); ++i) {
        const hp::HeOp& op = g->g.ops[i];
        if (op.ins.size() > AEGIS_MAX_OP_INPUTS) throw Error(AEGIS_EINVAL, "graph_export: op with too many operands");
        aegis_op_desc d{};
        d.kind = (uint32_t)op.kind;
        d.accumulate = op.accumulate;
        d.aligned = op.aligned;
        d.aggregation = (uint32_t)op.aggregation;
        d.rot_offset = op.rot_offset;
        d.phase = op.phase;
        d.out = aegis_slice{op.out.bundle, op.out.lane, op.out.lane_count};
        d.in_count = (uint32_t)op.ins.size();
        for (size_t k = 0; k < op.ins.size(); ++k) d.ins[k] = aegis_slice{op.ins[k].bundle, op.ins[k].lane, op.ins[k].lane_count};
        d.work = op.work;
        d.use_level = op.use_level;
        d.app_node = op.app_node;
        ops[i] = d;
      }
    if (inputs) std::copy(g->g.graph_inputs.begin(), g->g.graph_inputs.end(), inputs);
    if (n_inputs) *n_inputs = (uint32_t)g->g.graph_inputs.size();
    if (meta) {
      const uint64_t n = header_value(g->header, "N");
      aegis_graph_meta m{};
      while ((1ull << m.log_n) < n) ++m.log_n;
      m.chain_length = (uint32_t)header_value(g->header, "L");
      m.bootstrap_level = (uint32_t)header_value(g->header, "lboot");
      m.slots_per_token = (uint32_t)header_value(g->header, "stok");
      m.model_dim = (uint32_t)header_value(g->header, "d");
      m.head_dim = (uint32_t)header_value(g->header, "hd");
      m.ffn_dim = (uint32_t)header_value(g->header, "dff");
      m.layers = (uint32_t)header_value(g->header, "layers");
      m.kind = (uint32_t)header_value(g->header, "kind");
      m.tokens = header_value(g->header, "T");
      *meta = m;
    }
  });
}
int aegis_graph_set_shard(aegis_graph* g, uint32_t world, uint32_t rank) {
  if (!g) return AEGIS_EINVAL;
  return guard(nullptr, [&] {
    if (world <= 1) {
      g->shard.reset();
      return;
    }
    g->shard.reset(new aegis::ShardPlan(aegis::make_shard_plan(g->g, token_groups(g), world, rank)));
  });
}
int aegis_graph_set_hash_group(aegis_graph* g, int32_t group) {
  if (!g) return AEGIS_EINVAL;
  return guard(nullptr, [&] {
    if (group < 0) {
      g->hash_lanes.reset();
      return;
    }
    const uint32_t tg = token_groups(g);
    if ((uint32_t)group >= tg) throw Error(AEGIS_EINVAL, "token group out of range");
    g->hash_lanes.reset(new aegis::ShardPlan(aegis::make_shard_plan(g->g, tg, tg, (uint32_t)group)));
  });
}
int aegis_graph_set_reducer(aegis_graph* g, aegis_reduce_fn fn, void* user) {
  if (!g) return AEGIS_EINVAL;
  g->reduce = reinterpret_cast<aegis::ReduceFn>(fn);  // uint64_t* and u64* are the same 64-bit words
  g->reduce_user = user;
  return AEGIS_OK;
}
struct aegis_plan {
  aegis::ExecPlan p;
};
int aegis_plan_build(const aegis_graph* g, uint32_t world, int reorder, aegis_plan** out) {
  return guard(nullptr, [&] {
    if (!g || !out || world == 0) throw Error(AEGIS_EINVAL, "plan_build: bad argument");
    auto pl = std::make_unique<aegis_plan>();
    pl->p = aegis::build_plan(g->g, token_groups(g), world, (uint32_t)header_value(g->header, "N"), reorder != 0,
                              g->reference_modes != 0);
    *out = pl.release();
  });
}
int aegis_plan_summary_get(const aegis_plan* p, aegis_plan_summary* out) {
  if (!p || !out) return AEGIS_EINVAL;
  const aegis::ExecPlan& P = p->p;
  aegis_plan_summary s{};
  s.world = P.world;
  s.token_groups = P.tg_total;
  s.ranks_per_group = P.m;
  s.reordered = P.reordered;
  s.executable = P.executable;
  s.matmuls = (uint32_t)P.matmuls.size();
  s.events = P.events.size();
  for (const auto& d : P.devices) s.instrs_total += d.compute.size();
  for (const auto& e : P.events) {
    s.events_executed += e.executed;
    s.bytes_total += e.bytes_total;
    uint64_t* cat[] = {&s.bytes_ffn, &s.bytes_attention, &s.bytes_layernorm, &s.bytes_boot, &s.bytes_other};
    *cat[(int)e.category] += e.bytes_total;
  }
  for (const auto& m : P.matmuls) {
    s.matmuls_gather_chosen += m.chosen == aegis::MatmulMode::kGatherInputs;
    s.bytes_reference_rule += m.chosen == aegis::MatmulMode::kGatherInputs ? m.gather_bytes
                              : m.chosen == aegis::MatmulMode::kReduceOutputs ? m.reduce_bytes : 0;
  }
  *out = s;
  return AEGIS_OK;
}
int aegis_plan_events(const aegis_plan* p, aegis_plan_event* out, uint64_t cap, uint64_t* n) {
  if (!p || !n) return AEGIS_EINVAL;
  *n = p->p.events.size();
  if (out)
    for (uint64_t i = 0; i < std::min<uint64_t>(cap, *n); ++i) {
      const aegis::PlanEvent& e = p->p.events[i];
      out[i] = aegis_plan_event{e.id, (uint32_t)e.kind, (uint32_t)e.semantic, e.dev_lo, e.dev_count, e.bundle, e.lane,
                                e.lane_count, e.level, (uint32_t)e.category, e.app_node, e.he_op, e.executed,
                                e.bytes_per_device, e.bytes_total};
    }
  return AEGIS_OK;
}
int aegis_plan_device(const aegis_plan* p, uint32_t device, aegis_plan_instr* out, uint64_t cap, uint64_t* n) {
  if (!p || !n || device >= p->p.devices.size()) return AEGIS_EINVAL;
  const auto& C = p->p.devices[device].compute;
  *n = C.size();
  if (out)
    for (uint64_t i = 0; i < std::min<uint64_t>(cap, *n); ++i)
      out[i] = aegis_plan_instr{C[i].op, C[i].lane, C[i].lane_count, C[i].flags, C[i].wait_event};
  return AEGIS_OK;
}
int aegis_plan_matmuls(const aegis_plan* p, aegis_plan_matmul* out, uint64_t cap, uint64_t* n) {
  if (!p || !n) return AEGIS_EINVAL;
  *n = p->p.matmuls.size();
  if (out)
    for (uint64_t i = 0; i < std::min<uint64_t>(cap, *n); ++i) {
      const aegis::MatmulInfo& m = p->p.matmuls[i];
      out[i] = aegis_plan_matmul{m.app_node, m.acc_bundle, m.input_bundle, m.ship_bundle, (uint32_t)m.chosen,
                                 (uint32_t)m.executed, m.gather_bytes, m.reduce_bytes};
    }
  return AEGIS_OK;
}
const char* aegis_plan_note(const aegis_plan* p) { return p ? p->p.note.c_str() : ""; }
int aegis_graph_from_plan(const aegis_graph* g, const aegis_plan* p, uint32_t device, aegis_graph** out) {
  return guard(nullptr, [&] {
    if (!g || !p || !out) throw Error(AEGIS_EINVAL, "graph_from_plan: null argument");
    if (device >= p->p.devices.size()) throw Error(AEGIS_EINVAL, "graph_from_plan: no such device in the plan");
    const auto& C = p->p.devices[device].compute;
    std::vector<char> seen(g->g.ops.size(), 0);
    auto ng = std::make_unique<aegis_graph>();
    ng->g.bundles = g->g.bundles;
    ng->g.graph_inputs = g->g.graph_inputs;
    ng->header = g->header;
    for (const aegis::PlanInstr& in : C) {
      if (in.op >= g->g.ops.size()) throw Error(AEGIS_EINVAL, "graph_from_plan: plan does not belong to this graph");
      if (seen[in.op]) continue;
      seen[in.op] = 1;
      ng->g.ops.push_back(g->g.ops[in.op]);
    }
    for (size_t i = 0; i < seen.size(); ++i)  // ops the device runs no lane of keep their place at the end
      if (!seen[i]) ng->g.ops.push_back(g->g.ops[i]);
    hp::validate_heops(ng->g);
    *out = ng.release();
  });
}
int aegis_plan_free(aegis_plan* p) {
  delete p;
  return AEGIS_OK;
}
int aegis_graph_comm_bytes(const aegis_graph* g, uint64_t* bytes) {
  if (!g || !bytes) return AEGIS_EINVAL;
  *bytes = g->comm;
  return AEGIS_OK;
}
int aegis_graph_p2p_bytes(const aegis_graph* g, uint64_t* bytes) {
  if (!g || !bytes) return AEGIS_EINVAL;
  return guard(nullptr, [&] {
    uint64_t best = 0;
    const uint32_t m = g->shard ? g->shard->m : 1;
    if (m > 1) {
      const uint64_t n = header_value(g->header, "N");
      for (const hp::HeOp& op : g->g.ops) {
        if (op.kind != hp::HeOpKind::kPMult || op.ins.size() != 2) continue;
        const hp::CtBundle& acc = g->g.bundles[op.out.bundle];
        const aegis::PcmmShape sh = aegis::pcmm_shape(op.ins[0].lane_count, op.out.lane_count, op.ins[1].lane_count,
                                                      acc.chunk_period);
        const uint64_t share = sh.c_sub / m;
        best = std::max<uint64_t>(best, share * std::max<uint32_t>(2, acc.components) * acc.level * n);
        if (g->reference_modes) {  // the activation's share of a gather-mode matmul (up to 3 allocated comps)
          const hp::CtBundle& x = g->g.bundles[op.ins[0].bundle];
          best = std::max<uint64_t>(best, (uint64_t)(sh.c_in / m) * 3 * x.level * n);
        }
      }
    }
    *bytes = 2 * (uint64_t)m * best * 8;  // two parities x m slots x the largest share
  });
}
int aegis_graph_set_p2p(aegis_graph* g, aegis_p2p* w) {
  if (!g) return AEGIS_EINVAL;
  g->p2p = w ? w->w.get() : nullptr;
  return AEGIS_OK;
}
int aegis_graph_set_stored_weights(aegis_graph* g, int enable) {
  if (!g) return AEGIS_EINVAL;
  g->stored_weights = enable != 0;
  return AEGIS_OK;
}
int aegis_pmult_acc_stored(aegis_ctx* ctx, aegis_bundle* acc, uint32_t acc_lane, uint32_t acc_lanes,
                           uint32_t chunk_period, const aegis_bundle* x, uint32_t x_lane, uint32_t x_lanes,
                           const aegis_bundle* w, uint32_t w_lane, uint32_t w_lanes, uint32_t level) {
  return guard(ctx, [&] {
    Bundle& A = need(acc);
    const Bundle& X = need(x);
    const Bundle& W = need(w);
    check_lanes(A, acc_lane, acc_lanes, "pmult");
    check_lanes(X, x_lane, x_lanes, "pmult");
    check_lanes(W, w_lane, w_lanes, "pmult");
    check_level(A, level, "pmult");
    check_level(X, level, "pmult");
    check_level(W, level, "pmult");
    ctx->c->op_pmult(A, acc_lane, acc_lanes, chunk_period, X, x_lane, x_lanes, 0, w_lanes, level, 0, ~0u, 0, ~0u, &W,
                     w_lane);
  });
}
int aegis_graph_set_matmul_modes(aegis_graph* g, int reference_rule) {
  if (!g) return AEGIS_EINVAL;
  g->reference_modes = reference_rule != 0;
  return AEGIS_OK;
}
int aegis_graph_set_fault(aegis_graph* g, int kind) {
  if (!g || kind < 0 || kind > 1) return AEGIS_EINVAL;
  g->fault = kind;
  return AEGIS_OK;
}
int aegis_graph_owned_lanes(const aegis_graph* g, uint32_t bundle, uint8_t* mask, uint32_t cap) {
  if (!g || bundle >= g->g.bundles.size()) return AEGIS_EINVAL;
  const uint32_t lanes = g->g.bundles[bundle].lanes;
  for (uint32_t l = 0; l < lanes && l < cap; ++l) mask[l] = g->shard ? (g->shard->owns(bundle, l) ? 1 : 0) : 1;
  return AEGIS_OK;
}
int aegis_graph_shard_info(const aegis_graph* g, uint32_t* tg_total, uint32_t* tg_lo, uint32_t* tg_hi,
                           uint32_t* ranks_per_group, uint32_t* part) {
  if (!g) return AEGIS_EINVAL;
  const aegis::ShardPlan* s = g->shard.get();
  uint32_t tg = 1;
  try {
    tg = token_groups(g);
  } catch (...) {
  }
  if (tg_total) *tg_total = tg;
  if (tg_lo) *tg_lo = s ? s->tg_lo : 0;
  if (tg_hi) *tg_hi = s ? s->tg_hi : tg;
  if (ranks_per_group) *ranks_per_group = s ? s->m : 1;
  if (part) *part = s ? s->part : 0;
  return AEGIS_OK;
}
int aegis_graph_set_profiling(aegis_graph* g, int enable) {
  if (!g) return AEGIS_EINVAL;
  g->profile = enable != 0;
  return AEGIS_OK;
}
int aegis_graph_op_times(const aegis_graph* g, float* ms, uint64_t cap, uint64_t* n) {
  if (!g) return AEGIS_EINVAL;
  for (size_t i = 0; i < g->op_ms.size() && i < cap; ++i) ms[i] = g->op_ms[i];
  if (n) *n = g->op_ms.size();
  return AEGIS_OK;
}
int aegis_graph_comm_times(const aegis_graph* g, float* out, uint64_t cap, uint64_t* n) {
  if (!g) return AEGIS_EINVAL;
  const size_t k = g->comm_trace.size() / 3;
  for (size_t i = 0; i < k && i < cap && out; ++i)
    for (int j = 0; j < 3; ++j) out[3 * i + j] = g->comm_trace[3 * i + j];
  if (n) *n = k;
  return AEGIS_OK;
}
int aegis_graph_set_dce(aegis_graph* g, int enable) {
  if (!g) return AEGIS_EINVAL;
  g->dce = enable;
  return AEGIS_OK;
}
int aegis_graph_set_wrap_defer(aegis_graph* g, int enable) {
  if (!g) return AEGIS_EINVAL;
  g->wrap_defer = enable;
  return AEGIS_OK;
}
int aegis_graph_set_hoisting(aegis_graph* g, int enable) {
  if (!g) return AEGIS_EINVAL;
  g->hoist = enable;
  return AEGIS_OK;
}
int aegis_graph_io_bytes(const aegis_graph* g, uint64_t* h2d, uint64_t* d2h) {
  if (!g) return AEGIS_EINVAL;
  if (h2d) *h2d = g->h2d;
  if (d2h) *d2h = g->d2h;
  return AEGIS_OK;
}
int aegis_graph_key_ids(const aegis_graph* g, uint64_t* ids, uint32_t cap, uint32_t* n) {
  if (!g || !n) return AEGIS_EINVAL;
  std::set<uint64_t> s;
  for (const hp::HeOp& op : g->g.ops) {
    if (op.kind == hp::HeOpKind::kRot) {
      if (op.rot_offset <= -500) return AEGIS_EINVAL;  // validate_heops rejects these at load
      s.insert(1000u + (uint64_t)(int64_t)op.rot_offset);
    }
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
    aegis::RunOptions opt;
    opt.max_ops = max_ops;
    u64* dh = nullptr;
    if (hashes) {
      dh = c.alloc(nb);
      AEGIS_CHECK_CUDA(cudaMemsetAsync(dh, 0, nb * 8, c.stream));
      opt.d_hash = (unsigned long long*)dh;
    }
    run_graph(ctx, g, opt);
    if (hashes) {
      std::vector<u64> h(nb);
      AEGIS_CHECK_CUDA(cudaMemcpyAsync(h.data(), dh, nb * 8, cudaMemcpyDeviceToHost, c.stream));
      AEGIS_CHECK_CUDA(cudaStreamSynchronize(c.stream));
      for (size_t i = 0; i < nb && i < nhashes; ++i) hashes[i] = h[i];
      c.release(dh);
    }
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
    aegis::RunOptions opt;
    opt.host_in = reinterpret_cast<const u64*>(in);
    opt.host_out = reinterpret_cast<u64*>(out);
    run_graph(ctx, g, opt);
    AEGIS_CHECK_CUDA(cudaStreamSynchronize(c.stream));
  });
}
int aegis_graph_free(aegis_graph* g) {
  delete g;
  return AEGIS_OK;
}
uint64_t aegis_graph_peak_bytes(const aegis_graph* g) { return g ? g->peak : 0; }


int aegis_p2p_create(aegis_ctx* ctx, uint64_t bytes, void* handle_out, aegis_p2p** out) {
  if (!ctx || !handle_out || !out) return AEGIS_EINVAL;
  return guard(ctx, [&] {
    auto* h = new aegis_p2p;
    try {
      h->w.reset(aegis::p2p_create(*ctx->c, bytes, handle_out));
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}
int aegis_p2p_open(aegis_ctx* ctx, aegis_p2p* w, const void* handles, uint32_t m, uint32_t self) {
  if (!ctx || !w || !handles) return AEGIS_EINVAL;
  return guard(ctx, [&] { aegis::p2p_open(*w->w, handles, m, self); });
}
int aegis_p2p_open_local(aegis_ctx* ctx, aegis_p2p* w, aegis_p2p* const* group, uint32_t m, uint32_t self) {
  if (!ctx || !w || !group) return AEGIS_EINVAL;
  return guard(ctx, [&] {
    std::vector<aegis::P2pWindow*> v;
    for (uint32_t r = 0; r < m; ++r) v.push_back(group[r] ? group[r]->w.get() : nullptr);
    aegis::p2p_open_local(*w->w, v, self);
  });
}
int aegis_p2p_stage(aegis_ctx* ctx, aegis_p2p* w, const uint64_t* buf, uint64_t words) {
  if (!ctx || !w || !buf) return AEGIS_EINVAL;
  return guard(ctx, [&] { aegis::p2p_stage(*ctx->c, *w->w, reinterpret_cast<const aegis::u64*>(buf), words); });
}
int aegis_p2p_reduce(aegis_ctx* ctx, aegis_p2p* w, uint64_t* dst, uint64_t words_per_rank, uint32_t part) {
  if (!ctx || !w || !dst) return AEGIS_EINVAL;
  return guard(ctx, [&] { aegis::p2p_reduce(*ctx->c, *w->w, reinterpret_cast<aegis::u64*>(dst), words_per_rank, part); });
}
int aegis_p2p_destroy(aegis_p2p* w) {
  delete w;
  return AEGIS_OK;
}

}  // extern "C"

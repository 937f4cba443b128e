// kernels.h -- launch wrappers for the non-NTT kernels of libaegis.
#pragma once
#include "common.cuh"

namespace aegis {

// A strided view of a bundle: element (lane, comp, limb, x) lives at
// base + ((lane * comps + comp) * levels + limb) * n + x
struct View {
  u64* base;
  u32 lanes, comps, levels;
  __host__ __device__ u64* limb(u32 lane, u32 comp, u32 lb, u32 n) const {
    return base + (((size_t)lane * comps + comp) * levels + lb) * n;
  }
};

// Lane selection of one operand (he_ir.hpp:200-222 emit_per_lane rule):
// output lane l reads lane0 + (count == nout ? l : l % count).
struct LaneMap {
  u32 lane0, count;
  __host__ __device__ u32 at(u32 l, u32 nout) const { return lane0 + (count == nout ? l : l % count); }
};

constexpr int kMaxConv = 64;  // max source or target limbs of one conversion
constexpr int kMaxBigWords = 28;

// Exact centred basis-conversion constants (rns_math.hpp:151-193 restated at
// production size).  Device resident.
struct ConvPlanDev {
  u32 k, m;
  u64 src_p[kMaxConv], src_mu[kMaxConv];
  u64 hat_inv[kMaxConv], hat_inv_p[kMaxConv];   // (B/b_i)^{-1} mod b_i + Shoup
  u64 w_hi[kMaxConv], w_lo[kMaxConv];           // floor(2^128 / b_i)
  u64 dst_p[kMaxConv], dst_mu[kMaxConv];
  u64 b_mod[kMaxConv];                          // B mod d_t
  u64 dst_mu96[kMaxConv];                       // floor(2^96 / d_t): lazy reduction in ntt.cu cfwd_a
  u32 big_words;
  u64 b_big[kMaxBigWords];                      // B (multiword, little endian)
  // followed in memory by: hat_mod[k][m], hat_mod_p[k][m], hat_big[k][big_words]
};

struct ConvIO {
  const u64* src;  // source lane base (coefficient domain)
  size_t src_lane_stride;
  u32 src_off[kMaxConv];  // limb offsets (in units of n) of the k sources
  u64* dst;
  size_t dst_lane_stride;
  u32 dst_off[kMaxConv];  // limb offsets of the m targets
};

cudaError_t launch_basis_convert(const ConvPlanDev* plan, const u64* hat_tables, const ConvIO& io,
                                 u32 lanes, u32 n, u32 k, u32 m, cudaStream_t st);

// conversion prep (k <= 4): sources -> xt in place, overflow counts -> vbuf[lane * v_ls + x];
// both written in 24-bit split form (low 24 bits | high bits << 32) for cfwd_a's MACs
cudaError_t launch_conv_prep(const ConvPlanDev* plan, const u64* hat_tables, const ConvIO& io, u64* vbuf,
                             size_t v_ls, u32 lanes, u32 n, u32 k, u32 m, cudaStream_t st);

// rows of a view filled with the DESIGN.md §2.3 PRNG:
// row key = row_key(seed, tag, a, lane, comp, limb) for every (lane, comp, limb)
cudaError_t launch_fill_uniform(View v, u32 lanes, u32 comps, u32 limbs, u32 n, u64 seed, u64 tag,
                                u64 a, const u32* limb_ext, const PrimeConst* pc, cudaStream_t st);

// key tensor [digit][comp][slot][n], slot -> ext prime via slot_ext
cudaError_t launch_fill_key(u64* key, u32 digits, u32 slots, u32 n, u64 seed, u64 key_id,
                            const u32* slot_ext, const PrimeConst* pc, cudaStream_t st);

// eval-domain automorphism (rns_math.hpp:127-139, §8(a) A5): out = in[idx(j)]
cudaError_t launch_automorphism(View out, LaneMap om, View in, LaneMap im, u32 nlanes, u32 comps,
                                u32 limbs, u32 log_n, u64 galois, cudaStream_t st);

// out[l] = a[ma(l)] (x) b[mb(l)] tensor product (CMult, poly_ir.hpp:53): 3 comps
cudaError_t launch_cmult(View out, u32 out_lane0, View a, LaneMap ma, View b, LaneMap mb, u32 nlanes,
                         u32 limbs, u32 n, const PrimeConst* pc, cudaStream_t st);

// CAdd: acc ? out[l] += a[ma(l)] : out[l] = a[ma(l)] + b[mb(l)]   (2 comps)
cudaError_t launch_cadd(View out, u32 out_lane0, View a, LaneMap ma, View b, LaneMap mb, bool acc,
                        u32 nlanes, u32 comps, u32 limbs, u32 n, const PrimeConst* pc, cudaStream_t st);

// Bundled PCMM step (he_ir.hpp:360-371):
// acc[t*c_out+o] += sum_ci X[t*c_in+ci] * W[ci*c_out+o], W generated in-kernel.
// acc lane (t, o) = acc_lane0 + t*acc_tstride + o ; X lane (t, ci) = x_lane0 + t*x_tstride + ci ;
// weight lane = (ci_off + ci) * w_cout + o_off + o   (t < tg, ci < c_in, o < c_out)
struct PmultArgs {
  View acc;
  u32 acc_lane0, acc_tstride;
  View x;
  u32 x_lane0, x_tstride;
  u32 tg, c_in, c_out, ci_off, o_off, w_cout, limbs, n;
  const u64* rowkeys;
  // stored-plaintext variant: when wst.base is
  // set the weights are read from this 1-component bundle (lane = weight lane
  // + w_lane0) instead of being generated in-kernel; rowkeys is then unused
  View wst{nullptr, 0, 1, 0};
  u32 w_lane0 = 0;
};
cudaError_t launch_pmult_acc(const PmultArgs& a, const PrimeConst* pc, cudaStream_t st);
cudaError_t launch_weight_rowkeys(u64* out, u32 wlanes, u32 limbs, u64 seed, u64 bundle,
                                  cudaStream_t st);

// key inner product (poly_ir.hpp:264-275): for every lane and ext slot t
//   acc_c[t] = sum_j e_j[t] * key[j][c][keyslot(t)],  e_j[t] = d[t] when t in D_j
struct KeyMulIO {
  const u64* ext;        // [lane][digit][slot][n]
  size_t ext_lane_stride;
  const u64* d;          // original polynomial (NTT domain), [limb][n] per lane
  size_t d_lane_stride;
  u64* acc;              // [lane][comp][slot][n]
  size_t acc_lane_stride;
  const u64* key;        // [digit][comp][keyslot][n]
  u32 key_slots;         // chain + 4
  u32 level, dnum, nslots;   // nslots = level + 4
  u32 ext_lazy;              // ext words are lazy FP64 bits (NttLaunch::lazy_out), F64 path only
  u32 slot_ext[kMaxConv + 8];  // ext prime of slot
  u32 slot_key[kMaxConv + 8];  // key slot of slot
};
extern int g_km_f64;  // key product on the DFMA pipe (AEGIS_KM_F64=0: 24-bit integer MACs)
cudaError_t launch_keymul(const KeyMulIO& io, u32 lanes, u32 n, const PrimeConst* pc, cudaStream_t st);

// ModDown / rescale finish: out_c[i] = add_c[i] + (x_c[i] - y_c[i]) * f_i mod q_i
struct FinishIO {
  const u64* x; size_t x_lane, x_comp;
  const u64* y; size_t y_lane, y_comp;
  const u64* add; size_t add_lane, add_comp;  // may be null
  u64* out; size_t out_lane, out_comp;
  u32 comps, limbs;
  u64 galois;  // 1: none; else out[t] = f(inputs at pi_galois(t)) (eval-domain automorphism)
  u32 log_n;
  u32 ext[kMaxConv];
  u64 f[kMaxConv], f_p[kMaxConv];
};
cudaError_t launch_finish(const FinishIO& io, u32 lanes, u32 n, const PrimeConst* pc, cudaStream_t st);

// strided limb copy: lanes x comps x limbs rows of n words; source limbs start at src_limb0
cudaError_t launch_copy(View dst, u32 dst_lane0, View src, LaneMap sm, u32 nlanes, u32 comps, u32 limbs,
                        u32 src_limb0, u32 n, cudaStream_t st);

// DESIGN.md §2.4 content hash over lanes x comps x limbs (dense positions)
// (lanes [lane0, lane0+lanes) only; positions use absolute lane indices so shard
// hashes sum to the unsharded hash)
cudaError_t launch_hash(View v, u32 lane0, u32 lanes, u32 comps, u32 limbs, u32 n, unsigned long long* out,
                        cudaStream_t st);
cudaError_t launch_reduce_lanes(View v, u32 lane0, u32 lanes, u32 comps, u32 limbs, u32 n, const PrimeConst* pc,
                                cudaStream_t st);

// pointwise limb instruction (limb_ops.cu; opcode = LimbOpcode, poly_ir.hpp:49-58) over
// lanes x limbs [limb_lo, limb_lo + limbs) of every output component
cudaError_t launch_limb_op(int opcode, View out, u32 out_lane0, u32 out_comps, View a, LaneMap ma, u32 a_comps,
                           View b, LaneMap mb, u32 b_comps, u32 nlanes, u32 limb_lo, u32 limbs, u32 n,
                           const PrimeConst* pc, cudaStream_t st);
// kGenerate rows keyed by (seed, tag, bundle, absolute lane, comp, absolute limb)
cudaError_t launch_limb_generate(View out, u32 out_lane0, u32 nlanes, u32 comps, u32 limb_lo, u32 limbs, u32 n,
                                 u64 seed, u64 tag, u64 bundle, const PrimeConst* pc, cudaStream_t st);

}  // namespace aegis

// ntt.h -- launch descriptor for the batched NTT (see ntt.cu).
#pragma once

#include <vector>
#include "common.cuh"

namespace aegis {

struct PrimeTw {
  const ulonglong2* fwd;  // N entries (w, shoup(w)) : psi^brv(i)   (rns_math.hpp:59)
  const ulonglong2* inv;  // N entries : psi^-brv(i)                 (rns_math.hpp:60)
  const double2* fwd64;   // N entries (w, w/p) as doubles (FP64 butterflies)
  const double2* inv64;
  const double* fw;       // N entries w as doubles (v2 passes: w/p is formed at use)
  const double* iw;
  const double* fb;       // N = 2^16 only: pass-B twiddle blobs per tile (see ntt.cu v2)
  const double* ib;
  u64 p;
};
struct NttScale {
  u64 n_inv, n_inv_p;  // N^{-1} mod p and its Shoup companion (rns_math.hpp:62, 99)
  u64 w1n, w1n_p;      // inv[1] * N^{-1}: last GS stage with the scale folded in
  u64 mu64;            // floor(2^64 / p): one-step reduction of lazy values
  double pd, pinv;     // p and 1/p as doubles
  double n_inv_d, n_inv_wp, w1n_d, w1n_wp;  // FP64 forms of the scale constants
};

// Butterfly arithmetic of the NTT passes.
enum NttImpl : int { kNttInt = 0, kNttF64 = 1 };
extern int g_ntt_impl;  // selected at context creation (AEGIS_NTT_IMPL=int|f64)
extern int g_ntt_v2;      // N = 2^16 FP64 passes with direct global access (AEGIS_NTT_V2=0 disables)
extern int g_conv_fused;  // fused conversion + NTT (AEGIS_CONV_FUSED=0 disables)
extern int g_km_split;    // non-hoisted KS: ModUp pass B fused into the key product (AEGIS_KM_SPLIT=0 disables)

constexpr int kMaxSlots = 96;

// A batch of limbs ("rows"): row r -> lane r / nslots, slot r % nslots,
// address base + lane*lane_stride + slot_off[slot]*n, prime ext index prime[slot].
struct NttLaunch {
  u64* base;
  size_t lane_stride;
  u32 nlanes, nslots, n;
  u32 slot_off[kMaxSlots];
  unsigned char prime[kMaxSlots];
  const PrimeTw* tw;       // device, indexed by ext prime
  const NttScale* scale;   // device, indexed by ext prime
  // optional out-of-place input of the first inverse pass (v2 only):
  // row (lane, slot) reads in_base + lane*in_lane_stride + in_slot_off[slot]*n
  const u64* in_base;
  size_t in_lane_stride;
  u32 in_slot_off[kMaxSlots];
  // forward (v2): leave the outputs lazy (raw FP64 bits, |x| < 2^51, congruent
  // to the result) instead of canonical u64 -- for ModUp outputs that only the
  // FP64 key product reads
  u32 lazy_out;
};

// pass-B twiddle blob of one 16-sub tile at N = 2^16 (ntt.cu v2):
// per sub 15 rows x 17 doubles of round-2 twiddles + 15 round-1 twiddles
constexpr int kNttBlobSub = 15 * 17 + 15;
constexpr int kNttBlobTile = 16 * kNttBlobSub;
// build the fwd (or inv) blob of one prime from its bit-reversed power table tab[0..2^16)
void ntt_build_blob(const double* tab, double* blob);

// Fused exact basis conversion + forward NTT (N = 2^16, k <= 4 sources): the
// targets of L (slot s = conversion target s) are computed from the prepared
// sources (launch_conv_prep: xt_i in place, overflow counts v) as
//   y = sum_i xt_i [B/b_i]_t + v (t - [B]_t)  mod t
// inside the first NTT pass, so the converted limbs never round-trip HBM.
struct ConvPlanDev;
struct NttConvIn {
  const ConvPlanDev* plan;
  const u64* hat_tab;  // [k][m] (B/b_i) mod t
  const u64* src;      // prepared sources, coefficient domain
  size_t src_ls;
  u32 src_off[4];
  u32 k;
  const u64* v;        // overflow counts [lane][n]
  size_t v_ls;
};
// Optional epilogue of the second forward pass (ModDown / rescale finish):
// for virtual lane vl = lane * comps + comp and slot i of the launch,
//   z[s]  = (x[s] - y[s]) * f_i  (+ add[s] when comp < add_comps)
//   out[t] = z[s] at t = s (galois_inv <= 1) or t = pi_{galois_inv}(s)
// where y is the NTT output; y itself is never written to HBM.
struct NttFin {
  const u64* x;  long long x_lane, x_comp;
  const u64* add; long long add_lane, add_comp;
  u64* out; long long out_lane, out_comp;
  u32 comps, add_comps;
  u64 galois, galois_inv;  // galois_inv <= 1: no automorphism
  u32 log_n;
  u64 f[kMaxSlots];
};
cudaError_t ntt_conv_fwd(const NttLaunch& L, const NttConvIn& c, const NttFin* fin, cudaStream_t st,
                         bool pass_a_only = false);
// plain forward NTT with the finish epilogue (sources already converted)
cudaError_t ntt_fwd_fin(const NttLaunch& L, const NttFin& fin, cudaStream_t st);

// Second forward pass of the ModUp NTTs fused with the key inner product
// (non-hoisted key switching): for slot t of `lane`, each digit's pass-A
// intermediate (compact ModUp layout, written by ntt_conv_fwd with pass_a_only)
// is finished in registers and multiplied into the two key components;
// acc[lane][c][t] = sum_j E_j(t) * key[j][c][t] is the only output.
struct KmB {
  const u64* ext; size_t ext_ls;  // pass-A intermediates, lazy FP64 bits
  const u64* d; size_t d_ls;      // own-digit limbs (NTT domain, canonical)
  const u64* key;                 // [digit][comp][keyslot][n]
  u64* acc; size_t acc_ls;        // [lane][comp][slot][n]
  const PrimeTw* tw;
  const NttScale* scale;
  u32 key_slots, level, dnum, nslots, chain, nlanes, n;
};
cudaError_t ntt_fwd_b_keymul(const KmB& k, cudaStream_t st);

// true when ntt_run uses the v2 passes (out-of-place inverse, fused epilogues available)
bool ntt_v2_active(int log_n);

cudaError_t ntt_run(const NttLaunch& L, int log_n, bool inverse, cudaStream_t st);

// Kernel probe (measurement only: bench.py's roofline of the step's top
// kernels).  While g_probe is set, CUDA events bracket every launch of the
// probed kernel class on its stream and its algorithmic bytes (DESIGN.md §3:
// each input read once, each output written once) are summed.
enum ProbeKind { kProbeOff = 0, kProbeCfwdA = 1, kProbeFwdBFin = 2, kProbeFwdBKm = 3 };
struct KernelProbe {
  int kind = kProbeOff;
  std::vector<cudaEvent_t> ev;  // begin/end pairs
  double alg_bytes = 0;
  uint64_t launches = 0;
};
extern KernelProbe* g_probe;

}  // namespace aegis

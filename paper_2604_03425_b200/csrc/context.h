// context.h -- internal C++ state behind the aegis_* C-ABI.
#pragma once

#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/aegis.h"
#include "arena.h"
#include "kernels.h"
#include "ntt.h"
#include "shard.h"

namespace aegis {

// Error carrying an AEGIS_E* code across the C++ layer (mapped at the C-ABI).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
#define AEGIS_CHECK_CUDA(expr)                                                          \
  do {                                                                                  \
    cudaError_t e__ = (expr);                                                           \
    if (e__ != cudaSuccess)                                                             \
      throw ::aegis::Error(AEGIS_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e__)); \
  } while (0)

struct Plan {  // device-resident basis conversion constants
  ConvPlanDev* dev = nullptr;
  u64* tables = nullptr;
  u32 k = 0, m = 0;
};

struct Bundle {
  u64* ptr = nullptr;
  u32 lanes = 0, comps = 0, level = 0;
  size_t bytes = 0;
  View view() const { return View{ptr, lanes, comps, level}; }
};

class Context {
 public:
  Context(const aegis_params& p, int device);
  ~Context();

  // parameters
  u32 log_n, n, chain, lboot;
  u64 seed_input, seed_weight, seed_key;
  int device;
  cudaStream_t stream = nullptr, comm = nullptr;
  u64 launches = 0;

  u64 prime(u32 e) const { return primes_.at(e); }
  u32 post_boot_level() const { return chain - lboot; }

  // device tables
  PrimeConst* d_pc = nullptr;  // [kNumExt]
  PrimeTw* d_tw = nullptr;     // [kNumExt]
  NttScale* d_scale = nullptr; // [kNumExt]
  u32* d_ident = nullptr;      // identity limb -> ext map [0..kNumExt)

  // memory (stream ordered)
  u64* alloc(size_t words);
  void release(void* p);
  // return idle pool / arena memory to the device (synchronises the stream)
  void trim();
  static constexpr size_t kArenaMin = (size_t)4 << 20;  // allocations >= this come from the arena
  size_t live_bytes = 0, peak_bytes = 0;

  Bundle* new_bundle(u32 lanes, u32 comps, u32 level, bool zero);
  void free_bundle(Bundle* b);

  // basis conversion plans
  const Plan& plan(const std::vector<u32>& src_ext, const std::vector<u32>& dst_ext);

  // keys
  void generate_key(u64 key_id);
  void upload_key(u64 key_id, const u64* host, size_t words, bool coeff_domain);
  const u64* key(u64 key_id);
  // device storage of key `key_id` in the internal (pre-permuted) layout:
  // the existing key, or a fresh uninitialised one (store.cu loads into it)
  u64* key_storage(u64 key_id, bool create);
  void drop_key(u64 key_id);
  // fingerprint of the prime chain (main + special): files written under a
  // different chain are rejected (store.cu)
  u64 chain_fingerprint() const;
  u32 key_slots() const { return chain + kAlpha; }
  u32 key_digits() const { return (chain + kAlpha - 1) / kAlpha; }
  size_t key_bytes() const { return (size_t)key_digits() * 2 * key_slots() * n * 8; }
  size_t total_key_bytes() const { return keys_.size() * key_bytes(); }

  // ---- polynomial instructions --------------------------------------------
  // NTT over rows: lanes x slots, slot_off[i] limbs into the lane, primes[i]
  // src (inverse, v2 only): read the input from src + lane*src_ls + src_off[slot]*n
  // (src_off defaults to slot_off) and write the result to base
  void ntt(u64* base, size_t lane_stride, u32 nlanes, const std::vector<u32>& slot_off,
           const std::vector<u32>& primes, bool inverse, const u64* src = nullptr, size_t src_ls = 0,
           const std::vector<u32>* src_off = nullptr);
  void basis_convert(const u64* src, size_t src_lane_stride, const std::vector<u32>& src_off,
                     const std::vector<u32>& src_ext, u64* dst, size_t dst_lane_stride,
                     const std::vector<u32>& dst_off, const std::vector<u32>& dst_ext, u32 lanes);
  // exact conversion + forward NTT of the targets (fused at N = 2^16, k <= 4);
  // clobbers the sources; vbuf: lanes * n words of scratch.  With `fin` the
  // finish epilogue is fused into the last pass when the fused path runs
  // (returns true); otherwise dst holds the NTT and the caller finishes.
  bool conv_ntt(u64* src, size_t src_lane_stride, const std::vector<u32>& src_off, const std::vector<u32>& src_ext,
                u64* dst, size_t dst_lane_stride, const std::vector<u32>& dst_off, const std::vector<u32>& dst_ext,
                u32 lanes, u64* vbuf, const NttFin* fin = nullptr, bool lazy_out = false, bool pass_a_only = false);
  // ModUp outputs are left lazy (FP64 bits) when the fused conversion and the
  // FP64 key product are both active: the key product is their only reader
  bool modup_lazy() const {
    return log_n == 16 && g_ntt_impl == kNttF64 && g_ntt_v2 && g_conv_fused && g_km_f64;
  }
  // Hybrid key switch (poly_ir.hpp:219-298) of `lanes` polynomials d (level
  // limbs each, NTT domain, lane stride d_ls).  out_c = add_c + KS_c(d).
  struct KsOut {
    u64* out[2];
    size_t out_lane[2];
    const u64* add[2];
    size_t add_lane[2];
  };
  // galois != 1 applies the eval-domain automorphism to the result (Rot with
  // pre-permuted rotation keys).
  void keyswitch(const u64* d, size_t d_ls, u32 lanes, u32 level, u64 key_id, const KsOut& o, u64 galois = 1);
  struct KsShape {
    u32 l, ns, dn;
  };
  KsShape ks_shape(u32 l) const;
  // compact ModUp output: digit j holds its ns - |D_j| converted slots, at
  // word offset (j * ns - first prime of D_j) * n  (own-digit slots are read from d)
  size_t modup_words_per_lane(u32 l) const { return ((size_t)ks_shape(l).dn * ks_shape(l).ns - l) * n; }
  // ext[lane][digit][compact slot][n] = Ntt(exact lift of Intt(d) digit j to slot t)
  // pass_a_only: leave each digit's first-pass intermediate in ext (for ks_core(ext_pass_a))
  void modup(const u64* d, size_t d_ls, u32 lanes, u32 level, u64* ext, bool pass_a_only = false);
  void ks_core(const u64* ext, const u64* d, size_t d_ls, u32 lanes, u32 level, const u64* key, u64 galois,
               const KsOut& o, bool ext_pass_a = false);
  u64 galois_of(int offset) const;
  // key id of rotation r (poly_ir.hpp:300-305: 1000 + r).  Ids >= 500 mark
  // rotation keys (stored pre-permuted), so offsets <= -500 are rejected.
  static u64 rotation_key_id(int offset) {
    if (offset <= -500) throw Error(AEGIS_EINVAL, "rotation offset must be > -500 (key id 1000 + r)");
    return 1000u + (u64)(long long)offset;
  }

  // ---- HE operators --------------------------------------------------------
  void op_rot(Bundle& out, u32 out_lane, const Bundle& in, LaneMap im, u32 lanes, u32 level, int offset);
  void op_rot_cached(Bundle& out, u32 out_lane, const Bundle& in, LaneMap im, u32 lanes, u32 level, int offset,
                     const u64* ext);
  void op_relin(Bundle& b, u32 lane, u32 lanes, u32 level);
  void op_rescale(Bundle& out, u32 out_lane, const Bundle& in, LaneMap im, u32 lanes, u32 level);
  void op_boot(Bundle& out, u32 out_lane, const Bundle& in, LaneMap im, u32 lanes, u32 level, u32 out_level);
  void op_cmult(Bundle& out, u32 out_lane, u32 lanes, const Bundle& a, LaneMap ma, const Bundle& b,
                LaneMap mb, u32 level);
  void op_cadd(Bundle& out, u32 out_lane, u32 lanes, const Bundle& a, LaneMap ma, const Bundle* b,
               LaneMap mb, u32 level, bool acc);
  // token groups [t_lo, t_hi) and input positions [ci_lo, ci_hi) of the PCMM
  // step (defaults: everything); a position subset yields partial sums.
  void op_pmult(Bundle& acc, u32 acc_lane, u32 acc_lanes, u32 chunk_period, const Bundle& x, u32 x_lane,
                u32 x_lanes, u32 wbundle, u32 wlanes, u32 level, u32 t_lo = 0, u32 t_hi = ~0u, u32 ci_lo = 0,
                u32 ci_hi = ~0u, const Bundle* wstored = nullptr, u32 w_lane0 = 0, u32 o_lo = 0,
                u32 o_cnt = ~0u);  // outputs [o_lo, o_lo + o_cnt) of every sub-tensor

  void count(u64 k = 1) { launches += k; }
  // workspace budget of one operator phase: `gib` GiB scaled by AEGIS_WS_SCALE
  // (bigger lane batches = fewer, fuller launches; more scratch memory)
  size_t ws_budget(size_t gib) const { return (size_t)((double)(gib << 30) * ws_scale); }
  double ws_scale = 3.0;
  std::string last_error;

 private:
  std::vector<u64> primes_;
  u64* d_twiddles_ = nullptr;
  double* d_twd_ = nullptr;  // w-only FP64 twiddles [ext][fwd|inv][n]
  double* d_blob_ = nullptr; // N = 2^16 pass-B twiddle blobs [ext][fwd|inv][16 tiles]
  std::map<std::vector<u32>, Plan> plans_;
  std::map<u64, u64*> keys_;
  u32* d_key_slot_ext_ = nullptr;  // key slot -> ext prime
  u64* alloc_key();
  void prepermute_key(u64 key_id, u64* k);
  cudaMemPool_t pool_ = nullptr;
  std::unique_ptr<Arena> arena_;
};

}  // namespace aegis

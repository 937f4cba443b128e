// ntt.h -- launch descriptor for the batched NTT (see ntt.cu).
#pragma once
#include "common.cuh"

namespace aegis {

struct PrimeTw {
  const ulonglong2* fwd;  // N entries (w, shoup(w)) : psi^brv(i)   (rns_math.hpp:59)
  const ulonglong2* inv;  // N entries : psi^-brv(i)                 (rns_math.hpp:60)
  u64 p;
};
struct NttScale {
  u64 n_inv, n_inv_p;  // N^{-1} mod p and its Shoup companion (rns_math.hpp:62, 99)
  u64 w1n, w1n_p;      // inv[1] * N^{-1}: last GS stage with the scale folded in
  u64 mu64;            // floor(2^64 / p): one-step reduction of lazy values
};

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
};

cudaError_t ntt_run(const NttLaunch& L, int log_n, bool inverse, cudaStream_t st);

}  // namespace aegis

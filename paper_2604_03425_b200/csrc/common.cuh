// common.cuh -- shared device/host definitions for libaegis (sm_100a).
//
// Modular arithmetic for primes p < 2^48 (include/aegis_params.h) on 64-bit
// words.  Semantics follow rns_math.hpp:21-40 (canonical results in [0, p));
// the implementations are B200-specific:
//   * Shoup multiplication by a precomputed constant (twiddles, CRT factors):
//     one __umul64hi + two 64-bit mul.lo, result in [0, 2p) then one
//     conditional subtract.
//   * data x data products are accumulated as u128 and reduced once with a
//     Barrett step valid for sums < 2^104 (up to 256 products of 48-bit
//     residues) -- see reduce104().
#pragma once

#include <cstdint>
#include <utility>
#include <cuda_runtime.h>

#include "../../include/aegis_params.h"

namespace aegis {

using u64 = unsigned long long;
using u32 = unsigned int;

constexpr u32 kSpecialBase = AEGIS_MAX_MAIN_PRIMES;  // ext index of P_0
constexpr u32 kNumExt = AEGIS_MAX_MAIN_PRIMES + AEGIS_SPECIAL_PRIMES;
constexpr u32 kAlpha = AEGIS_SPECIAL_PRIMES;  // digit width of hybrid key switching
constexpr u64 kGold = 0x9E3779B97F4A7C15ULL;
constexpr u64 kMixM = 0xD6E8FEB86659FD93ULL;

// Per-prime constants (device resident, indexed by ext prime index).
struct PrimeConst {
  u64 p;
  u64 mu104;   // floor(2^104 / p) for reduce104
  u32 shift;   // 64 - bitlen(p): PRNG -> [0, 2p) mapping
  u32 pad;
};

struct u128 {
  u64 lo, hi;
};

__host__ __device__ __forceinline__ u64 mix64(u64 x) {
  x ^= x >> 32;
  x *= kMixM;
  x ^= x >> 32;
  x *= kMixM;
  x ^= x >> 32;
  return x;
}

// DESIGN.md §2.3 counter PRNG: row key per (seed, tag, a, b, c, d).
__host__ __device__ __forceinline__ u64 row_key(u64 seed, u64 tag, u64 a, u64 b, u64 c, u64 d) {
  u64 k = mix64(seed ^ (tag * kGold));
  k = mix64(k ^ ((a + 1) * kGold));
  k = mix64(k ^ ((b + 1) * kGold));
  k = mix64(k ^ ((c + 1) * kGold));
  k = mix64(k ^ ((d + 1) * kGold));
  return k;
}

__host__ __device__ __forceinline__ u64 uniform_at(u64 rk, u64 i, u64 p, u32 shift) {
  u64 v = mix64(rk + i * kGold) >> shift;
  return v >= p ? v - p : v;
}

#ifdef __CUDACC__

__device__ __forceinline__ u64 add_mod(u64 a, u64 b, u64 p) {
  u64 s = a + b;
  return s >= p ? s - p : s;
}
__device__ __forceinline__ u64 sub_mod(u64 a, u64 b, u64 p) {
  return a >= b ? a - b : a + p - b;
}
// a * w mod p with wp = floor(w 2^64 / p); valid for any a < 2^64.
__device__ __forceinline__ u64 shoup_lazy(u64 a, u64 w, u64 wp, u64 p) {
  const u64 q = __umul64hi(a, wp);
  return a * w - q * p;  // in [0, 2p)
}
__device__ __forceinline__ u64 shoup(u64 a, u64 w, u64 wp, u64 p) {
  const u64 r = shoup_lazy(a, w, wp, p);
  return r >= p ? r - p : r;
}

__device__ __forceinline__ u128 mul_wide(u64 a, u64 b) {
  u128 r;
  r.lo = a * b;
  r.hi = __umul64hi(a, b);
  return r;
}
__device__ __forceinline__ void mac(u128& acc, u64 a, u64 b) {
  const u64 lo = a * b;
  const u64 hi = __umul64hi(a, b);
  acc.lo += lo;
  acc.hi += hi + (acc.lo < lo ? 1 : 0);
}
__device__ __forceinline__ void add_to(u128& acc, u64 a) {
  acc.lo += a;
  acc.hi += (acc.lo < a ? 1 : 0);
}
// s < 2^104  ->  s mod p  (p in (2^42, 2^48)).  q_est = floor((s >> 40) mu / 2^64)
// is within 3 of floor(s / p) from below.
__device__ __forceinline__ u64 reduce104(u128 s, u64 p, u64 mu) {
  const u64 top = (s.lo >> 40) | (s.hi << 24);
  const u64 q = __umul64hi(top, mu);
  u64 r = s.lo - q * p;
  r = r >= p ? r - p : r;
  r = r >= p ? r - p : r;
  r = r >= p ? r - p : r;
  return r;
}
__device__ __forceinline__ u64 mul_mod(u64 a, u64 b, u64 p, u64 mu) {
  return reduce104(mul_wide(a, b), p, mu);
}

// ---- multiply-accumulate on 24-bit limbs ------------------------------------
// Residues are < 2^48, so a = a1 2^24 + a0 with a0, a1 < 2^24 and every limb
// product is < 2^48: each column accumulates 2^16 products in a u64 without a
// carry, and one MAC is four IMAD.WIDE.U32 (vs ~12 instructions for a
// 64x64->128 multiply plus 128-bit add).
struct Split {
  u32 lo, hi;
};
__device__ __forceinline__ Split split24(u64 a) { return Split{(u32)(a & 0xFFFFFFu), (u32)(a >> 24)}; }

struct Acc3 {
  u64 c0 = 0, c1 = 0, c2 = 0;  // value = c0 + c1 2^24 + c2 2^48
};
__device__ __forceinline__ void mac24(Acc3& s, Split a, Split b) {
  s.c0 += (u64)a.lo * b.lo;
  s.c1 += (u64)a.lo * b.hi;
  s.c1 += (u64)a.hi * b.lo;
  s.c2 += (u64)a.hi * b.hi;
}
// the same MAC as four mad.wide.u32 in PTX.  Only for pmult_kernel: there it
// removes a zero-add per product (-20% time), while in the NTT-fused
// conversion (cfwd_a) the PTX form made ptxas schedule worse (+18% key switch)
__device__ __forceinline__ void mad_wide(u64& acc, u32 a, u32 b) {
  asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc) : "r"(a), "r"(b));
}
__device__ __forceinline__ void mac24_ptx(Acc3& s, Split a, Split b) {
  mad_wide(s.c0, a.lo, b.lo);
  mad_wide(s.c1, a.lo, b.hi);
  mad_wide(s.c1, a.hi, b.lo);
  mad_wide(s.c2, a.hi, b.hi);
}
__device__ __forceinline__ u128 acc3_value(const Acc3& s) {
  u128 r;
  r.lo = s.c0 + (s.c1 << 24);
  u64 carry = r.lo < s.c0 ? 1 : 0;
  r.hi = (s.c1 >> 40) + carry;
  const u64 t = s.c2 << 48;
  r.lo += t;
  r.hi += (r.lo < t ? 1 : 0) + (s.c2 >> 16);
  return r;
}
// sum < 2^104 (<= 256 products of 48-bit residues) -> canonical residue
__device__ __forceinline__ u64 acc3_reduce(const Acc3& s, u64 p, u64 mu) { return reduce104(acc3_value(s), p, mu); }

// 256-bit global accesses (sm_100: LDG/STG.E.ENL2.256), 32-byte aligned
__device__ __forceinline__ void ld256g(const u64* p, u64& a, u64& b, u64& c, u64& d) {
  asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}
__device__ __forceinline__ void st256g(u64* p, u64 a, u64 b, u64 c, u64 d) {
  asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}

// read-only, no L1 allocation (data shared across CTAs through L2 only)
__device__ __forceinline__ void ld256na(const u64* p, u64& a, u64& b, u64& c, u64& d) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
               : "l"(p));
}

// programmatic dependent launch: block until the preceding grid in the stream
// has completed and its writes are visible (a no-op for ordinary launches)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// cache prefetches (no registers, no completion tracking)
__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// streaming (evict-first) variants for data touched once per kernel
__device__ __forceinline__ void ld256cs(const u64* p, u64& a, u64& b, u64& c, u64& d) {
  asm volatile("ld.global.cs.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}
__device__ __forceinline__ void st256cs(u64* p, u64 a, u64 b, u64 c, u64 d) {
  asm volatile("st.global.cs.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}

// ---- exact FP64 modular arithmetic (p < 2^46; see ntt.cu v2 for the bounds) ----
constexpr double kF64Magic = 6755399441055744.0;  // 1.5 * 2^52: round on the DFMA pipe
constexpr double kF64Two52 = 4503599627370496.0;
__device__ __forceinline__ double f64_of(u64 x) {  // exact for x < 2^52
  return __longlong_as_double((long long)(x | 0x4330000000000000ULL)) - kF64Two52;
}
// y * w mod p in [-1.5p, 1.5p] for |y * w / p| < 2^51, wp ~ w / p
__device__ __forceinline__ double f64_mulmod(double y, double w, double wp, double p) {
  const double h = y * w;
  const double l = fma(y, w, -h);
  const double q = fma(y, wp, kF64Magic) - kF64Magic;
  return fma(-q, p, h) + l;
}
// |x| < 2^51 -> canonical residue
__device__ __forceinline__ u64 f64_canon(double x, double p, double pinv) {
  const double r = fma(-((x * pinv + kF64Magic) - kF64Magic), p, x);  // integer in (-p, p)
  // range corrections on the integer pipe (r + 1.5 * 2^52 carries r in its mantissa)
  const long long pi = __double_as_longlong(p + kF64Two52) & 0xFFFFFFFFFFFFFLL;
  long long y = __double_as_longlong(r + kF64Magic) - 0x4338000000000000LL;
  y = y < 0 ? y + pi : y;
  y = y >= pi ? y - pi : y;
  return (u64)y;
}

extern int g_pdl;  // programmatic dependent launch of the key-switch kernels (AEGIS_PDL)

// launch with the programmatic-stream-serialization attribute: the grid may be
// scheduled while its predecessor drains; the kernel must pdl_wait() before it
// touches any data an earlier kernel produces or consumes
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

#endif  // __CUDACC__

}  // namespace aegis

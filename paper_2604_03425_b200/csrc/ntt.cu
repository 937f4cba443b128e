// ntt.cu -- batched negacyclic NTT / INTT for sm_100a.
//
// Semantics: exactly NegacyclicNtt::forward / ::inverse of rns_math.hpp:68-100
// (Cooley-Tukey DIT, natural order in -> bit-reversed evaluation order out;
// Gentleman-Sande inverse followed by the N^{-1} scale, which we fold into the
// last GS stage).  psi and the bit-reversed twiddle tables are the
// reference's (rns_math.hpp:53-61, 103-117), built on the host in context.cu.
// Outputs are canonical residues, so any exact butterfly arithmetic gives
// bit-identical results.
//
// B200 design: an N = 2^(kA+kB) transform is two passes over
// HBM, each a batch of small SMEM-resident sub-transforms:
//   pass A  -- the first kA stages act on the 2^kB "columns" j = c + 2^kB u
//              (stride-2^kB sub-problems).  A CTA stages 16 adjacent columns
//              (128-byte coalesced row segments) in shared memory;
//   pass B  -- the last kB stages act on contiguous blocks of 2^kB.
// Inside a CTA each thread owns 2^R elements of one sub-problem in registers
// and runs R butterfly stages per shared-memory round trip (radix-2^R); the
// SMEM layout pads one word per 16 (+1 per sub-problem) so both the strided
// and the contiguous round patterns are bank-conflict free.
//
// Two butterfly implementations (g_ntt_impl):
//   kNttInt -- 64-bit Shoup with lazy (Harvey) reduction.  Bound by the
//              IMAD pipe: ~13 IMAD-class instructions per butterfly.
//   kNttF64 -- exact FP64 modular multiply: h = y*w, l = fma(y,w,-h) (exact
//              product split), q = rint(y * w/p), r = fma(-q,p,h) + l.  With
//              primes < 2^46 every intermediate is an integer < 2^52, so the
//              arithmetic is exact; it runs on the DFMA pipe (58.5/clk/SM on
//              B200) and leaves the integer pipes to addressing.
// The intermediate between the two passes is lazy (raw u64 or raw double bits);
// only values leaving the transform are canonicalised.
#include <cstring>
#include <type_traits>

#include "kernels.h"
#include "ntt.h"

namespace aegis {

int g_ntt_impl = kNttF64;
int g_ntt_v2 = 1;
int g_conv_fused = 1;
int g_pdl = 1;
int g_km_split = 1;

namespace {

__device__ __forceinline__ u32 pad_idx(u32 u) { return u + (u >> 4); }

constexpr int radix_for(int logm) {
  return logm == 8 ? 4 : logm == 9 ? 3 : logm == 6 ? 3 : logm == 5 ? 5 : logm == 4 ? 4
       : logm == 3 ? 3 : logm == 2 ? 2 : 1;
}

template <int LOGM>
struct SubCfg {
  static constexpr int R = radix_for(LOGM);
  static constexpr int M = 1 << LOGM;
  static constexpr int TPS = 1 << (LOGM - R);    // threads per sub-problem
  static constexpr int STRIDE = M + M / 16 + 1;  // padded SMEM words per sub-problem
  static constexpr int ROUNDS = LOGM / R;
  static_assert(LOGM % R == 0, "radix must divide the sub-transform size");
};

struct RowInfo {
  u64* ptr;
  u32 prime;
};

__device__ __forceinline__ RowInfo row_info(const NttLaunch& L, u32 row) {
  const u32 lane = row / L.nslots;
  const u32 slot = row - lane * L.nslots;
  RowInfo r;
  r.ptr = L.base + (size_t)lane * L.lane_stride + (size_t)L.slot_off[slot] * L.n;
  r.prime = L.prime[slot];
  return r;
}

// ---------------------------------------------------------------------------
// integer butterflies (lazy Harvey: p < 2^46 leaves >= 18 bits of headroom)
// ---------------------------------------------------------------------------
__device__ __forceinline__ u64 reduce_lazy(u64 x, u64 p, u64 mu) {
  const u64 r = x - __umul64hi(x, mu) * p;  // in [0, 2p)
  return r >= p ? r - p : r;
}

struct IntArith {
  using T = u64;
  using Tw = ulonglong2;
  u64 p, two_p;
  const NttScale* sc;
  __device__ __forceinline__ void ct(T& a, T& b, Tw w) const {
    const u64 t = shoup_lazy(b, w.x, w.y, p);
    const u64 x = a;
    a = x + t;
    b = x + two_p - t;
  }
  // `bound` = 2^depth p: both inputs are below it
  __device__ __forceinline__ void gs(T& a, T& b, Tw w, u64 bound) const {
    const u64 x = a, y = b;
    a = x + y;
    b = shoup_lazy(x + bound - y, w.x, w.y, p);
  }
  __device__ __forceinline__ void gs_scale(T& a, T& b, u64 bound) const {
    const u64 x = a, y = b;
    a = shoup(x + y, sc->n_inv, sc->n_inv_p, p);
    b = shoup(x + bound - y, sc->w1n, sc->w1n_p, p);
  }
  __device__ __forceinline__ void round_end_gs(T&) const {}
  __device__ __forceinline__ T load_canon(u64 v) const { return v; }
  __device__ __forceinline__ T load_lazy(u64 v, bool inverse) const {
    return inverse ? reduce_lazy(v, p, sc->mu64) : v;
  }
  __device__ __forceinline__ u64 store_lazy(T v) const { return v; }
  __device__ __forceinline__ u64 store_canon(T v, bool already) const {
    return already ? v : reduce_lazy(v, p, sc->mu64);
  }
};

// ---------------------------------------------------------------------------
// FP64 butterflies: values are integer-valued doubles, |x| < 2^52
// ---------------------------------------------------------------------------
constexpr double kTwo52 = 4503599627370496.0;

__device__ __forceinline__ double u2d(u64 x) {  // exact for x < 2^52
  return __longlong_as_double((long long)(x | 0x4330000000000000ULL)) - kTwo52;
}
// y * w mod p as a value in about [-p/2 - 1, p/2 + 1]  (exact integer arithmetic)
__device__ __forceinline__ double mulmod_f64(double y, double w, double wp, double p) {
  const double h = y * w;
  const double l = fma(y, w, -h);
  const double q = rint(y * wp);
  return fma(-q, p, h) + l;
}
// same, rounding with the 1.5 * 2^52 magic constant on the DFMA pipe (no XU
// FRND); valid while |y * w / p| < 2^51 -- true for the forward transform,
// whose lazy values stay below ~25 p < 2^51 with p < 2^46.
__device__ __forceinline__ double mulmod_f64_fast(double y, double w, double wp, double p) {
  constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
  const double h = y * w;
  const double l = fma(y, w, -h);
  const double q = fma(y, wp, kMagic) - kMagic;
  return fma(-q, p, h) + l;
}
__device__ __forceinline__ double reduce_f64(double x, double p, double pinv) {
  return fma(-rint(x * pinv), p, x);  // |result| <= p/2 + 1
}
__device__ __forceinline__ u64 canon_f64(double x, double p, double pinv) {
  double r = reduce_f64(x, p, pinv);
  r = r < 0.0 ? r + p : r;
  r = r >= p ? r - p : r;
  return (u64)__double_as_longlong(r + kTwo52) & 0xFFFFFFFFFFFFFULL;
}

struct F64Arith {
  using T = double;
  using Tw = double2;
  double p, pinv;
  const NttScale* sc;
  __device__ __forceinline__ void ct(T& a, T& b, Tw w) const {
    const double t = mulmod_f64_fast(b, w.x, w.y, p);
    const double x = a;
    a = x + t;
    b = x - t;
  }
  __device__ __forceinline__ void gs(T& a, T& b, Tw w, u64) const {
    const double x = a, y = b;
    a = x + y;
    b = mulmod_f64(x - y, w.x, w.y, p);
  }
  __device__ __forceinline__ void gs_scale(T& a, T& b, u64) const {
    const double x = a, y = b;
    a = mulmod_f64(x + y, sc->n_inv_d, sc->n_inv_wp, p);
    b = mulmod_f64(x - y, sc->w1n_d, sc->w1n_wp, p);
  }
  // the GS sum path doubles per stage: fold back below p once per round
  __device__ __forceinline__ void round_end_gs(T& x) const { x = reduce_f64(x, p, pinv); }
  __device__ __forceinline__ T load_canon(u64 v) const { return u2d(v); }
  __device__ __forceinline__ T load_lazy(u64 v, bool) const { return __longlong_as_double((long long)v); }
  __device__ __forceinline__ u64 store_lazy(T v) const { return (u64)__double_as_longlong(v); }
  __device__ __forceinline__ u64 store_canon(T v, bool) const { return canon_f64(v, p, pinv); }
};

// One radix-2^R round of forward CT stages s0 .. s0+R-1 on the sub-problem at sp.
template <int LOGM, class A>
__device__ __forceinline__ void ct_round(typename A::T* sp, u32 tau, int s0, u32 t0,
                                         const typename A::Tw* __restrict__ tw, const A& ar) {
  using C = SubCfg<LOGM>;
  constexpr int R = C::R;
  const int lo_bits = LOGM - s0 - R;
  const u32 tau_lo = tau & ((1u << lo_bits) - 1);
  const u32 tau_hi = tau >> lo_bits;
  const u32 base = tau_lo | (tau_hi << (lo_bits + R));
  // issue every twiddle load of the round up front (2^R - 1 independent
  // 128-bit loads in flight) instead of one dependent load per butterfly
  typename A::Tw wv[(1 << R) - 1];
#pragma unroll
  for (int sg = 0; sg < R; ++sg)
#pragma unroll
    for (int q = 0; q < (1 << sg); ++q) wv[(1 << sg) - 1 + q] = tw[(t0 << (s0 + sg)) + (tau_hi << sg) + q];
  typename A::T x[1 << R];
#pragma unroll
  for (int v = 0; v < (1 << R); ++v) x[v] = sp[pad_idx(base | ((u32)v << lo_bits))];
#pragma unroll
  for (int sg = 0; sg < R; ++sg) {
    const int half = 1 << (R - sg - 1);
#pragma unroll
    for (int v = 0; v < (1 << R); ++v) {
      if (v & half) continue;
      ar.ct(x[v], x[v + half], wv[(1 << sg) - 1 + (v >> (R - sg))]);
    }
  }
#pragma unroll
  for (int v = 0; v < (1 << R); ++v) sp[pad_idx(base | ((u32)v << lo_bits))] = x[v];
}

// One radix-2^R round of inverse GS stages s0+R-1 .. s0 (descending).  `depth`
// counts GS stages since values were last reduced (integer bounds).  When
// `last` is set the round contains the global final stage (s == 0 of pass A):
// there N^{-1} is folded into both outputs.
template <int LOGM, class A>
__device__ __forceinline__ void gs_round(typename A::T* sp, u32 tau, int s0, u32 t0,
                                         const typename A::Tw* __restrict__ tw, const A& ar, int depth,
                                         bool last, u64 p) {
  using C = SubCfg<LOGM>;
  constexpr int R = C::R;
  const int lo_bits = LOGM - s0 - R;
  const u32 tau_lo = tau & ((1u << lo_bits) - 1);
  const u32 tau_hi = tau >> lo_bits;
  const u32 base = tau_lo | (tau_hi << (lo_bits + R));
  typename A::Tw wv[(1 << R) - 1];  // all twiddle loads of the round in flight at once
#pragma unroll
  for (int sg = 0; sg < R; ++sg)
#pragma unroll
    for (int q = 0; q < (1 << sg); ++q)
      if (!(last && s0 + sg == 0)) wv[(1 << sg) - 1 + q] = tw[(t0 << (s0 + sg)) + (tau_hi << sg) + q];
  typename A::T x[1 << R];
#pragma unroll
  for (int v = 0; v < (1 << R); ++v) x[v] = sp[pad_idx(base | ((u32)v << lo_bits))];
#pragma unroll
  for (int sg = R - 1; sg >= 0; --sg) {
    const int s = s0 + sg;
    const int half = 1 << (R - sg - 1);
    const u64 bound = p << (depth + (R - 1 - sg));
    const bool scale = last && s == 0;
#pragma unroll
    for (int v = 0; v < (1 << R); ++v) {
      if (v & half) continue;
      if (scale) ar.gs_scale(x[v], x[v + half], bound);
      else ar.gs(x[v], x[v + half], wv[(1 << sg) - 1 + (v >> (R - sg))], bound);
    }
  }
  if (!last) {
#pragma unroll
    for (int v = 0; v < (1 << R); ++v) ar.round_end_gs(x[v]);
  }
#pragma unroll
  for (int v = 0; v < (1 << R); ++v) sp[pad_idx(base | ((u32)v << lo_bits))] = x[v];
}

// MODE 0: columns (pass A), MODE 1: contiguous blocks (pass B).
//   forward : pass A (canonical -> lazy), pass B (lazy -> canonical)
//   inverse : pass B (canonical -> lazy), pass A (lazy -> canonical)
template <int LOGM, int MODE, bool INV, int IMPL>
__global__ void __launch_bounds__(256, 3) ntt_pass_kernel(const NttLaunch L, int kA, int kB,
                                                       int subs_per_cta, int scale_last) {
  using C = SubCfg<LOGM>;
  using A = typename std::conditional<IMPL == kNttF64, F64Arith, IntArith>::type;
  using T = typename A::T;
  extern __shared__ u64 smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);
  const u32 ctas_per_row = MODE == 0 ? (1u << kB) / subs_per_cta : (1u << kA) / subs_per_cta;
  const u32 row = blockIdx.x / ctas_per_row;
  const u32 chunk = blockIdx.x - row * ctas_per_row;
  const RowInfo ri = row_info(L, row);
  const PrimeTw pt = L.tw[ri.prime];
  const NttScale* sc = L.scale + ri.prime;
  A ar;
  if constexpr (IMPL == kNttF64) {
    ar.p = sc->pd;
    ar.pinv = sc->pinv;
  } else {
    ar.p = pt.p;
    ar.two_p = 2 * pt.p;
  }
  ar.sc = sc;
  const typename A::Tw* __restrict__ tw;
  if constexpr (IMPL == kNttF64) tw = INV ? pt.inv64 : pt.fwd64;
  else tw = INV ? pt.inv : pt.fwd;
  const u32 nthreads = blockDim.x;
  const u32 total = subs_per_cta * C::M;
  // which side of this pass is canonical (the other is the lazy intermediate)
  const bool in_canon = (!INV && MODE == 0) || (INV && MODE == 1);

  // ---- load (coalesced) ----
  if (MODE == 0) {
    const u32 c0 = chunk * subs_per_cta;
    const u32 cmask = subs_per_cta - 1;
    const int clog = __ffs(subs_per_cta) - 1;
    for (u32 e = threadIdx.x; e < total; e += nthreads) {
      const u32 c = e & cmask, u = e >> clog;
      const u64 v = ri.ptr[c0 + c + ((size_t)u << kB)];
      smem[c * C::STRIDE + pad_idx(u)] = in_canon ? ar.load_canon(v) : ar.load_lazy(v, INV);
    }
  } else {
    const size_t off = (size_t)chunk * total;
    for (u32 e = threadIdx.x; e < total; e += nthreads) {
      const u32 b = e >> LOGM, v = e & (C::M - 1);
      const u64 x = ri.ptr[off + e];
      smem[b * C::STRIDE + pad_idx(v)] = in_canon ? ar.load_canon(x) : ar.load_lazy(x, INV);
    }
  }
  __syncthreads();

  const u32 sub = threadIdx.x / C::TPS;
  const u32 tau = threadIdx.x - sub * C::TPS;
  T* sp = smem + sub * C::STRIDE;
  const u32 t0 = MODE == 0 ? 1u : (1u << kA) + chunk * subs_per_cta + sub;
  // block = subs_per_cta * TPS threads exactly, so every thread owns work
  if (!INV) {
#pragma unroll
    for (int rd = 0; rd < C::ROUNDS; ++rd) {
      ct_round<LOGM, A>(sp, tau, rd * C::R, t0, tw, ar);
      if (rd + 1 < C::ROUNDS) {
        if (C::TPS > 32) __syncthreads(); else __syncwarp();
      }
    }
  } else {
#pragma unroll
    for (int rd = C::ROUNDS - 1; rd >= 0; --rd) {
      gs_round<LOGM, A>(sp, tau, rd * C::R, t0, tw, ar, (C::ROUNDS - 1 - rd) * C::R, scale_last && rd == 0, pt.p);
      if (rd > 0) {
        if (C::TPS > 32) __syncthreads(); else __syncwarp();
      }
    }
  }
  __syncthreads();

  // ---- store (coalesced) ----
  // canonical output side: forward pass B and inverse pass A (the integer
  // inverse is already canonical after the scaled stage)
  const bool out_canon = !in_canon;
  const bool int_already = INV;
  if (MODE == 0) {
    const u32 c0 = chunk * subs_per_cta;
    const u32 cmask = subs_per_cta - 1;
    const int clog = __ffs(subs_per_cta) - 1;
    for (u32 e = threadIdx.x; e < total; e += nthreads) {
      const u32 c = e & cmask, u = e >> clog;
      const T x = smem[c * C::STRIDE + pad_idx(u)];
      ri.ptr[c0 + c + ((size_t)u << kB)] = out_canon ? ar.store_canon(x, int_already) : ar.store_lazy(x);
    }
  } else {
    const size_t off = (size_t)chunk * total;
    for (u32 e = threadIdx.x; e < total; e += nthreads) {
      const u32 b = e >> LOGM, v = e & (C::M - 1);
      const T x = smem[b * C::STRIDE + pad_idx(v)];
      ri.ptr[off + e] = out_canon ? ar.store_canon(x, int_already) : ar.store_lazy(x);
    }
  }
}

template <int LOGM, int MODE, bool INV, int IMPL>
cudaError_t launch_pass(const NttLaunch& L, int kA, int kB, u32 rows, int scale_last, cudaStream_t st) {
  using C = SubCfg<LOGM>;
  const int nsub_total = MODE == 0 ? (1 << kB) : (1 << kA);
  int subs = 256 / C::TPS;
  if (subs > nsub_total) subs = nsub_total;
  if (subs < 1) subs = 1;
  const u32 ctas_per_row = nsub_total / subs;
  const size_t smem = (size_t)subs * C::STRIDE * sizeof(u64);
  auto kern = ntt_pass_kernel<LOGM, MODE, INV, IMPL>;
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  const dim3 grid(rows * ctas_per_row);
  const dim3 block(subs * C::TPS);
  kern<<<grid, block, smem, st>>>(L, kA, kB, subs, scale_last);
  return cudaGetLastError();
}

template <int MODE, bool INV, int IMPL>
cudaError_t dispatch_pass(int logm, const NttLaunch& L, int kA, int kB, u32 rows, int scale_last,
                          cudaStream_t st) {
  switch (logm) {
    case 1: return launch_pass<1, MODE, INV, IMPL>(L, kA, kB, rows, scale_last, st);
    case 2: return launch_pass<2, MODE, INV, IMPL>(L, kA, kB, rows, scale_last, st);
    case 3: return launch_pass<3, MODE, INV, IMPL>(L, kA, kB, rows, scale_last, st);
    case 4: return launch_pass<4, MODE, INV, IMPL>(L, kA, kB, rows, scale_last, st);
    case 5: return launch_pass<5, MODE, INV, IMPL>(L, kA, kB, rows, scale_last, st);
    case 6: return launch_pass<6, MODE, INV, IMPL>(L, kA, kB, rows, scale_last, st);
    case 7: return launch_pass<7, MODE, INV, IMPL>(L, kA, kB, rows, scale_last, st);
    case 8: return launch_pass<8, MODE, INV, IMPL>(L, kA, kB, rows, scale_last, st);
    case 9: return launch_pass<9, MODE, INV, IMPL>(L, kA, kB, rows, scale_last, st);
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------------------
// v2: N = 2^16 FP64 passes (256 x 256) with direct-to-register global access.
//
// A CTA owns 16 sub-transforms of 256 points; each of its 256 threads holds
// 16 elements and runs two radix-16 rounds (stages 0-3, 4-7) with one SMEM
// exchange between them.  The thread -> (sub, tau) mapping is chosen per pass
// so that the round whose element pattern is "tau + 16 v" (pass B) or whose
// sub index is the column (pass A) touches global memory directly with
// 128-byte coalesced rows: all 16 loads of a thread are independent and in
// flight together (no SMEM staging, one exposed latency per tile).  Only the
// forward pass-B store and the inverse pass-B load (pattern "16 tau + v" on
// contiguous memory) are staged through SMEM.  Rounding uses the 1.5 * 2^52
// magic constant everywhere (no XU FRND).  Row order is slot-major so CTAs
// running together share one prime's twiddle table in L2.
// ---------------------------------------------------------------------------
namespace v2 {

constexpr int kStride = 273;  // 256 + 16 + 1 padded words per sub-transform
#ifndef AEGIS_CONV_TARGETS
#define AEGIS_CONV_TARGETS 2
#endif
constexpr int kConvTargets = AEGIS_CONV_TARGETS;  // conversion targets per cfwd_a CTA
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
// Pass-B twiddle blob (built by ntt_build_blob, one contiguous block per tile
// so a single TMA bulk copy stages it): per sub, round-2 twiddles stored
// [sg][q][tau] in 17-word rows (the 16 threads of a sub read one row per
// (sg, q): conflict free), then the 15 round-1 twiddles (half-warp broadcast).
constexpr int kTwRow = 17;
__device__ __host__ __forceinline__ int tw2_off(int sg, int q) { return ((1 << sg) - 1 + q) * kTwRow; }
constexpr int kTw1 = 15 * kTwRow;

__device__ __forceinline__ double rnd(double x) { return (x + kMagic) - kMagic; }
// y * w mod p, exact, result in about [-1.5p, 1.5p] (q may be off by one: wp = w * (1/p))
__device__ __forceinline__ double mm(double y, double w, double wp, double p) {
  const double h = y * w;
  const double l = fma(y, w, -h);
  const double q = fma(y, wp, kMagic) - kMagic;
  return fma(-q, p, h) + l;
}
__device__ __forceinline__ double red(double x, double p, double pinv) { return fma(-rnd(x * pinv), p, x); }
// canonical residue: one FP64 reduction, then the two range corrections on
// the idle integer pipe (r + 1.5 * 2^52 carries the integer r, |r| < 2^51, in
// its low mantissa bits; the compare/select form cost 4 more FP64-pipe ops)
__device__ __forceinline__ u64 canon(double x, double p, double pinv) {
  const double r = red(x, p, pinv);  // integer-valued, in (-p, p)
  const long long pi = __double_as_longlong(p + kTwo52) & 0xFFFFFFFFFFFFFLL;
  long long y = __double_as_longlong(r + kMagic) - 0x4338000000000000LL;
  y = y < 0 ? y + pi : y;
  y = y >= pi ? y - pi : y;
  return (u64)y;
}

// Radix-16 rounds.  TW(sg, q) returns the twiddle of stage sg, group q.
template <class TW>
__device__ __forceinline__ void ct16(double (&x)[16], TW tw, double p, double pinv) {
#pragma unroll
  for (int sg = 0; sg < 4; ++sg) {
    const int half = 8 >> sg;
#pragma unroll
    for (int q = 0; q < (1 << sg); ++q) {
      const double2 wv = tw(sg, q, pinv);
#pragma unroll
      for (int j = 0; j < half; ++j) {
        const int v = q * 2 * half + j;
        const double t = mm(x[v + half], wv.x, wv.y, p);
        const double a = x[v];
        x[v] = a + t;
        x[v + half] = a - t;
      }
    }
  }
}

// GS stages sg = 3..0; SCALE folds N^{-1} into the stage with sg == 0
template <bool SCALE, class TW>
__device__ __forceinline__ void gs16(double (&x)[16], TW tw, double p, double pinv, const NttScale* sc) {
#pragma unroll
  for (int sg = 3; sg >= 0; --sg) {
    const int half = 8 >> sg;
#pragma unroll
    for (int q = 0; q < (1 << sg); ++q) {
      double2 wv = make_double2(0.0, 0.0);
      if (!(SCALE && sg == 0)) wv = tw(sg, q, pinv);
#pragma unroll
      for (int j = 0; j < half; ++j) {
        const int v = q * 2 * half + j;
        const double a = x[v], b = x[v + half];
        if (SCALE && sg == 0) {
          x[v] = mm(a + b, sc->n_inv_d, sc->n_inv_wp, p);
          x[v + half] = mm(a - b, sc->w1n_d, sc->w1n_wp, p);
        } else {
          x[v] = a + b;
          x[v + half] = mm(a - b, wv.x, wv.y, p);
        }
      }
    }
  }
}

// Rounds with the 15 twiddles of the round preloaded (w only, w/p formed at
// use): all loads of a round are issued together at its start, so only the
// first stage waits on them.
template <int S0>
__device__ __forceinline__ void load_w(double (&w)[15], const double* __restrict__ tw, u32 t0, u32 th) {
#pragma unroll
  for (int sg = 0; sg < 4; ++sg)
#pragma unroll
    for (int q = 0; q < (1 << sg); ++q) w[(1 << sg) - 1 + q] = __ldg(tw + (t0 << (S0 + sg)) + (th << sg) + q);
}
__device__ __forceinline__ void load_w_blob(double (&w)[15], const double* sp) {
#pragma unroll
  for (int sg = 0; sg < 4; ++sg)
#pragma unroll
    for (int q = 0; q < (1 << sg); ++q) w[(1 << sg) - 1 + q] = sp[((1 << sg) - 1 + q) * 17];
}
// pass-B round-1 twiddles of one sub from the blob (half-warp broadcast)
[[maybe_unused]] __device__ __forceinline__ void load_w_blob1(double (&w)[15], const double* sb) {
#pragma unroll
  for (int i = 0; i < 15; ++i) w[i] = sb[kTw1 + i];
}
// 0: round-1 twiddles from the w-only table, so the blob's TMA copy is only
// waited for before round 2 (measured 0.4-0.6 % faster key switches at the
// end of round 1; the blob wait was 12 % of fwd_b_fin's stall samples)
#ifndef AEGIS_BLOB_R1
#define AEGIS_BLOB_R1 0
#endif
// fwd_b_fin: L2 prefetch of the finish operands at tile start (-0.4..0.6 % per
// key switch; the same idea as an L1 prefetch of fwd_b_km's key words cost 5 %)
#ifndef AEGIS_FIN_PREFETCH
#define AEGIS_FIN_PREFETCH 1
#endif
#ifndef AEGIS_KM_EXT_CS
#define AEGIS_KM_EXT_CS 0
#endif
// fwd_b_fin finish operands: read once, no L1 allocation (-0.6..1.2 %)
#ifndef AEGIS_FIN_NA
#define AEGIS_FIN_NA 1
#endif
// fwd_b_km key words: read-only, shared across lanes through L2, no L1
// allocation (L1 is what the 2 x 102 KB SMEM leaves; the allocating loads
// thrashed it: -7 % Relin, -8 % non-hoisted Rot)
#ifndef AEGIS_KM_KEY_NA
#define AEGIS_KM_KEY_NA 1
#endif
struct WArr {
  const double* w;
  __device__ __forceinline__ double2 operator()(int sg, int q, double pinv) const {
    const double t = w[(1 << sg) - 1 + q];
    return make_double2(t, t * pinv);
  }
};

__device__ __forceinline__ double dbits(u64 v) { return __longlong_as_double((long long)v); }
__device__ __forceinline__ u64 bitsd(double v) { return (u64)__double_as_longlong(v); }

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void blob_init(u64* mbar) {
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
}
// thread 0: arm the mbarrier and start the TMA bulk copy of a tile's blob
__device__ __forceinline__ void blob_issue(u64* mbar, double* dst, const double* src) {
  if (threadIdx.x == 0) {
    const u32 bar = smem_u32(mbar);
    constexpr u32 bytes = (u32)(kNttBlobTile * sizeof(double));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
  }
}
__device__ __forceinline__ void blob_wait(u64* mbar, u32 parity) {
  const u32 bar = smem_u32(mbar);
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n @!P bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void st256(u64* p, u64 a, u64 b, u64 c, u64 d) {
  asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
__device__ __forceinline__ void ld256(const u64* p, u64& a, u64& b, u64& c, u64& d) {
  asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}

// ---- per-tile bodies ------------------------------------------------------
// A tile is 16 sub-transforms of one row (limb): pass A = 16 adjacent columns,
// pass B = 16 contiguous blocks of 256.
struct RowRef {
  u64* ptr;
  u32 prime;
};
__device__ __forceinline__ RowRef row_ref(const NttLaunch& L, u32 lane, u32 slot) {
  return RowRef{L.base + (size_t)lane * L.lane_stride + (size_t)L.slot_off[slot] * L.n, L.prime[slot]};
}

// forward pass A: columns c = chunk*16 + lo, thread tau = hi.  canonical in, lazy out.
template <int KB = 8>  // column stride 2^KB (N = 2^(8+KB))
__device__ __forceinline__ void tile_fwd_a(const NttLaunch& L, RowRef rr, u32 chunk, double* sm) {
  const double* tw = L.tw[rr.prime].fw;
  const NttScale* sc = L.scale + rr.prime;
  const double p = sc->pd, pinv = sc->pinv;
  const u32 lo = threadIdx.x & 15, hi = threadIdx.x >> 4;
  u64* col = rr.ptr + chunk * 16 + lo;
  double x[16], w[15];
  u64 raw[16];
#pragma unroll
  for (int v = 0; v < 16; ++v) raw[v] = col[(size_t)(hi + 16 * v) << KB];
  load_w<0>(w, tw, 1, 0);
#pragma unroll
  for (int v = 0; v < 16; ++v) x[v] = u2d(raw[v]);
  ct16(x, WArr{w}, p, pinv);
#pragma unroll
  for (int v = 0; v < 16; ++v) sm[lo * kStride + hi + 17 * v] = x[v];
  load_w<4>(w, tw, 1, hi);
  __syncthreads();
#pragma unroll
  for (int v = 0; v < 16; ++v) x[v] = sm[lo * kStride + 17 * hi + v];
  ct16(x, WArr{w}, p, pinv);
#pragma unroll
  for (int v = 0; v < 16; ++v) col[(size_t)(16 * hi + v) << KB] = bitsd(x[v]);
}

// forward pass A of one column chunk, input already in registers (lazy)
__device__ __forceinline__ void pass_a_body(double (&x)[16], const double* tw, double p, double pinv, double* sm,
                                            u64* col) {
  const u32 lo = threadIdx.x & 15, hi = threadIdx.x >> 4;
  double w[15];
  load_w<0>(w, tw, 1, 0);
  ct16(x, WArr{w}, p, pinv);
#pragma unroll
  for (int v = 0; v < 16; ++v) sm[lo * kStride + hi + 17 * v] = x[v];
  load_w<4>(w, tw, 1, hi);
  __syncthreads();
#pragma unroll
  for (int v = 0; v < 16; ++v) x[v] = sm[lo * kStride + 17 * hi + v];
  ct16(x, WArr{w}, p, pinv);
#pragma unroll
  for (int v = 0; v < 16; ++v) col[(size_t)(16 * hi + v) << 8] = bitsd(x[v]);
}

// fused exact conversion + forward pass A for T target slots slot0 .. slot0+nt-1
// of lane `lane`: every prepared source word (launch_conv_prep: x~_i and v in
// 24-bit split form) is read once from L2 and feeds all T targets,
//   S_t = sum_i x~_i [B/b_i]_t + v (t - [B]_t),
// lazily reduced into [0, 3t).  Target 0 stays in registers; targets 1.. are
// parked in this thread's private SMEM slots (`hand`) until their pass runs.
template <int K, int T>
__device__ __forceinline__ void tile_cfwd_a(const NttLaunch& L, const NttConvIn& C, u32 lane, u32 slot0, u32 nt,
                                            u32 chunk, double* sm, u64* hand) {
  const ConvPlanDev* pl = C.plan;
  const u32 m = pl->m;
  Split hs[T][K + 1];
  u64 dd[T], mu[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const u32 slot = slot0 + ((u32)t < nt ? t : 0);
    dd[t] = pl->dst_p[slot];
    mu[t] = pl->dst_mu96[slot];
#pragma unroll
    for (int i = 0; i < K; ++i) hs[t][i] = split24(__ldg(C.hat_tab + (size_t)i * m + slot));
    hs[t][K] = split24(dd[t] - pl->b_mod[slot]);
  }
  const u32 lo = threadIdx.x & 15, hi = threadIdx.x >> 4;
  const size_t col0 = (size_t)chunk * 16 + lo + ((size_t)hi << 8);
  const uint2* ps[K + 1];
#pragma unroll
  for (int i = 0; i < K; ++i)
    ps[i] = reinterpret_cast<const uint2*>(C.src + (size_t)lane * C.src_ls + (size_t)C.src_off[i] * (1u << 16) + col0);
  ps[K] = reinterpret_cast<const uint2*>(C.v + (size_t)lane * C.v_ls + col0);
  double x[16];
#pragma unroll
  for (int v = 0; v < 16; ++v) {
    uint2 w[K + 1];
#pragma unroll
    for (int i = 0; i <= K; ++i) w[i] = __ldg(ps[i] + (v << 12));
#pragma unroll
    for (int t = 0; t < T; ++t) {
      u64 r;
      if constexpr (K == 1) {
        // one source (rescale, boot from level 1): B = b_0, so [B/b_0]_t = 1 and
        // the lift is x~ + v (d - [b_0]_d) -- no products; S < 2^48
        const u64 S = (u64)w[0].x + ((u64)w[0].y << 24) +
                      (w[1].x ? (u64)hs[t][1].lo + ((u64)hs[t][1].hi << 24) : 0ull);
        const u64 q = __umul64hi(S >> 32, mu[t]);
        r = S - q * dd[t];
      } else {
        Acc3 a;
#pragma unroll
        for (int i = 0; i < K; ++i) mac24(a, Split{w[i].x, w[i].y}, hs[t][i]);
        // the overflow count v <= k has a zero high limb: two products, not four
        a.c0 += (u64)w[K].x * hs[t][K].lo;
        a.c1 += (u64)w[K].x * hs[t][K].hi;
        // q = floor((S >> 32) floor(2^96/d) / 2^64) is within 3 below S/d: r = S - q d in [0, 3d)
        const u64 top = (a.c2 << 16) + (a.c1 >> 8) + (a.c0 >> 32);
        const u64 q = __umul64hi(top, mu[t]);
        r = a.c0 + (a.c1 << 24) + (a.c2 << 48) - q * dd[t];
      }
      if (t == 0) x[v] = u2d(r);
      else hand[(size_t)(t - 1) * 4096 + v * 256 + threadIdx.x] = r;
    }
  }
#pragma unroll
  for (int t = 0; t < T; ++t) {
    if ((u32)t >= nt) break;
    const RowRef rr = row_ref(L, lane, slot0 + t);
    const NttScale* sc = L.scale + rr.prime;
    if (t > 0) {
      __syncthreads();  // sm (exchange rows) is reused by the next target
#pragma unroll
      for (int v = 0; v < 16; ++v) x[v] = u2d(hand[(size_t)(t - 1) * 4096 + v * 256 + threadIdx.x]);
    }
    pass_a_body(x, L.tw[rr.prime].fw, sc->pd, sc->pinv, sm, rr.ptr + chunk * 16 + lo);
  }
}

// forward pass B: block b = chunk*16 + hi (256 contiguous), tau = lo.  lazy in,
// canonical out (each thread writes its 16 contiguous outputs as 4 x 32 B).
// The caller has issued the tile's blob copy on `mbar`.
__device__ __forceinline__ void tile_fwd_b(const NttLaunch& L, RowRef rr, u32 chunk, double* sm, const double* stw,
                                           u64* mbar, u32 parity) {
  const NttScale* sc = L.scale + rr.prime;
  const double p = sc->pd, pinv = sc->pinv;
  const u32 lo = threadIdx.x & 15, hi = threadIdx.x >> 4;
  u64* blk = rr.ptr + (size_t)(chunk * 16 + hi) * 256;
  double x[16], w[15];
#pragma unroll
  for (int v = 0; v < 16; ++v) x[v] = dbits(blk[lo + 16 * v]);
  const double* sb = stw + hi * kNttBlobSub;
#if AEGIS_BLOB_R1
  blob_wait(mbar, parity);
  load_w_blob1(w, sb);
#else
  load_w<0>(w, L.tw[rr.prime].fw, 256 + chunk * 16 + hi, 0);
#endif
  ct16(x, WArr{w}, p, pinv);
  double* sp = sm + hi * kStride;
#pragma unroll
  for (int v = 0; v < 16; ++v) sp[lo + 17 * v] = x[v];
  __syncwarp();
#if !AEGIS_BLOB_R1
  blob_wait(mbar, parity);
#endif
  load_w_blob(w, sb + lo);
#pragma unroll
  for (int v = 0; v < 16; ++v) x[v] = sp[17 * lo + v];
  ct16(x, WArr{w}, p, pinv);
  u64* o = blk + 16 * lo;
  if (L.lazy_out) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      st256(o + 4 * k, bitsd(x[4 * k]), bitsd(x[4 * k + 1]), bitsd(x[4 * k + 2]), bitsd(x[4 * k + 3]));
    return;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
    st256(o + 4 * k, canon(x[4 * k], p, pinv), canon(x[4 * k + 1], p, pinv), canon(x[4 * k + 2], p, pinv),
          canon(x[4 * k + 3], p, pinv));
}

// forward pass B with the ModDown / rescale finish epilogue (see NttFin)
__device__ __forceinline__ void tile_fwd_b_fin(const NttLaunch& L, const NttFin& F, u32 lane_v, u32 slot, u32 chunk,
                                               double* sm, const double* stw, u64* mbar, u32 parity) {
  const RowRef rr = row_ref(L, lane_v, slot);
  const NttScale* sc = L.scale + rr.prime;
  const double p = sc->pd, pinv = sc->pinv;
  const u32 lo = threadIdx.x & 15, hi = threadIdx.x >> 4;
  u64* blk = rr.ptr + (size_t)(chunk * 16 + hi) * 256;
  // the finish factor is a dynamically indexed kernel parameter (an LDC that
  // stalled the epilogue): fetch it now, its latency hides under the NTT
  const u64 f_bits = F.f[slot];
#if AEGIS_FIN_PREFETCH
  {  // the finish operands (one 128-byte line per thread each) start moving to
     // L2 now, while the NTT pass runs
    const u32 lane = lane_v / F.comps, comp = lane_v - lane * F.comps;
    const size_t s0 = (size_t)chunk * 4096 + (hi << 8) + 16 * lo;
    prefetch_l2(F.x + (long long)lane * F.x_lane + (long long)comp * F.x_comp + (size_t)slot * L.n + s0);
    if (F.add && comp < F.add_comps)
      prefetch_l2(F.add + (long long)lane * F.add_lane + (long long)comp * F.add_comp + (size_t)slot * L.n + s0);
  }
#endif
  double x[16], w[15];
#pragma unroll
  for (int v = 0; v < 16; ++v) x[v] = dbits(blk[lo + 16 * v]);
#if AEGIS_BLOB_R1
  blob_wait(mbar, parity);
  load_w_blob1(w, stw + hi * kNttBlobSub);
#else
  load_w<0>(w, L.tw[rr.prime].fw, 256 + chunk * 16 + hi, 0);
#endif
  ct16(x, WArr{w}, p, pinv);
  double* sp = sm + hi * kStride;
#pragma unroll
  for (int v = 0; v < 16; ++v) sp[lo + 17 * v] = x[v];
  __syncwarp();
#if !AEGIS_BLOB_R1
  blob_wait(mbar, parity);
#endif
  load_w_blob(w, stw + hi * kNttBlobSub + lo);
#pragma unroll
  for (int v = 0; v < 16; ++v) x[v] = sp[17 * lo + v];
  ct16(x, WArr{w}, p, pinv);
  // epilogue
  const u32 lane = lane_v / F.comps, comp = lane_v - lane * F.comps;
  const u32 sl = (hi << 8) + 16 * lo;                   // this thread's first position inside the tile
  const size_t s0 = (size_t)chunk * 4096 + sl;          // ... inside the limb
  const double f = u2d(f_bits), fp = f * pinv;
  const bool has_add = F.add && comp < F.add_comps;
  const u64* xr = F.x + (long long)lane * F.x_lane + (long long)comp * F.x_comp + (size_t)slot * L.n + s0;
  const u64* ar = has_add ? F.add + (long long)lane * F.add_lane + (long long)comp * F.add_comp + (size_t)slot * L.n + s0
                          : nullptr;
  u64* orow = F.out + (long long)lane * F.out_lane + (long long)comp * F.out_comp + (size_t)slot * L.n;
  const bool permute = F.galois_inv > 1;
  u64* su = reinterpret_cast<u64*>(sm);  // permuted output staging: 4096 words of the tile
  if (permute) __syncthreads();          // every thread is done with the exchange rows
#pragma unroll
  for (int k = 0; k < 4; ++k) {  // 4 positions at a time keeps the live state small
    u64 xv[4];
#if AEGIS_FIN_NA
    ld256na(xr + 4 * k, xv[0], xv[1], xv[2], xv[3]);
#else
    ld256(xr + 4 * k, xv[0], xv[1], xv[2], xv[3]);
#endif
    double z[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) z[i] = mm(u2d(xv[i]) - x[4 * k + i], f, fp, p);
    if (has_add) {
#if AEGIS_FIN_NA
      ld256na(ar + 4 * k, xv[0], xv[1], xv[2], xv[3]);
#else
      ld256(ar + 4 * k, xv[0], xv[1], xv[2], xv[3]);
#endif
#pragma unroll
      for (int i = 0; i < 4; ++i) z[i] += u2d(xv[i]);
    }
    const u64 c0 = canon(z[0], p, pinv), c1 = canon(z[1], p, pinv), c2 = canon(z[2], p, pinv),
              c3 = canon(z[3], p, pinv);
    if (!permute) {
      st256(orow + s0 + 4 * k, c0, c1, c2, c3);
    } else {
      su[sl + 4 * k] = c0;
      su[sl + 4 * k + 1] = c1;
      su[sl + 4 * k + 2] = c2;
      su[sl + 4 * k + 3] = c3;
    }
  }
  if (permute) {
    // out[t] = z[pi(t)]: pi maps aligned 32-blocks onto aligned 32-blocks, so
    // the tile's 128 source blocks are 128 whole target blocks; each thread
    // gathers half a target block from SMEM and writes it with 256-bit stores.
    __syncthreads();
    const u32 mask = 2u * L.n - 1, sh = 32 - F.log_n;
    const u32 kf = (u32)(F.galois & mask), ki = (u32)(F.galois_inv & mask);
    const u32 sb = (u32)chunk * 4096 + (threadIdx.x >> 1) * 32;  // source block of this thread pair
    const u32 tb = (__brev(((((__brev(sb) >> sh) * 2 + 1) * ki & mask) - 1) >> 1) >> sh) & ~31u;
    const u32 t0 = tb + 16 * (threadIdx.x & 1);
    u64 w[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const u32 t = t0 + i;
      const u32 sidx = __brev(((((__brev(t) >> sh) * 2 + 1) * kf & mask) - 1) >> 1) >> sh;
      w[i] = su[sidx - (u32)chunk * 4096];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) st256(orow + t0 + 4 * k, w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
  }
}

// inverse pass B (first): canonical in (4 x 32 B per thread), lazy out.
__device__ __forceinline__ void tile_inv_b(const NttLaunch& L, RowRef rr, const u64* src_row, u32 chunk, double* sm,
                                           const double* stw, u64* mbar, u32 parity) {
  const NttScale* sc = L.scale + rr.prime;
  const double p = sc->pd, pinv = sc->pinv;
  const u32 lo = threadIdx.x & 15, hi = threadIdx.x >> 4;
  u64* blk = rr.ptr + (size_t)(chunk * 16 + hi) * 256;
  const u64* sblk = src_row + (size_t)(chunk * 16 + hi) * 256;
  u64 raw[16];
#pragma unroll
  for (int k = 0; k < 4; ++k) ld256(sblk + 16 * lo + 4 * k, raw[4 * k], raw[4 * k + 1], raw[4 * k + 2], raw[4 * k + 3]);
  double x[16];
#pragma unroll
  for (int v = 0; v < 16; ++v) x[v] = u2d(raw[v]);
  double w[15];
  blob_wait(mbar, parity);
  const double* sb = stw + hi * kNttBlobSub;
  load_w_blob(w, sb + lo);
  gs16<false>(x, WArr{w}, p, pinv, sc);
  double* sp = sm + hi * kStride;
#pragma unroll
  for (int v = 0; v < 16; ++v) sp[17 * lo + v] = red(x[v], p, pinv);
#if AEGIS_BLOB_R1
  load_w_blob1(w, sb);
#else
  load_w<0>(w, L.tw[rr.prime].iw, 256 + chunk * 16 + hi, 0);
#endif
  __syncwarp();
#pragma unroll
  for (int v = 0; v < 16; ++v) x[v] = sp[lo + 17 * v];
  gs16<false>(x, WArr{w}, p, pinv, sc);
#pragma unroll
  for (int v = 0; v < 16; ++v) blk[lo + 16 * v] = bitsd(red(x[v], p, pinv));
}

// inverse pass A (second): columns c = chunk*16 + lo, tau = hi; lazy in, canonical out, N^{-1} folded.
template <int KB = 8>
__device__ __forceinline__ void tile_inv_a(const NttLaunch& L, RowRef rr, u32 chunk, double* sm) {
  const NttScale* sc = L.scale + rr.prime;
  const double p = sc->pd, pinv = sc->pinv;
  const u32 lo = threadIdx.x & 15, hi = threadIdx.x >> 4;
  u64* col = rr.ptr + chunk * 16 + lo;
  double x[16], w[15];
#pragma unroll
  for (int v = 0; v < 16; ++v) x[v] = dbits(col[(size_t)(16 * hi + v) << KB]);
  load_w<4>(w, L.tw[rr.prime].iw, 1, hi);
  gs16<false>(x, WArr{w}, p, pinv, sc);
#pragma unroll
  for (int v = 0; v < 16; ++v) sm[lo * kStride + 17 * hi + v] = red(x[v], p, pinv);
  load_w<0>(w, L.tw[rr.prime].iw, 1, 0);
  __syncthreads();
#pragma unroll
  for (int v = 0; v < 16; ++v) x[v] = sm[lo * kStride + hi + 17 * v];
  gs16<true>(x, WArr{w}, p, pinv, sc);
#pragma unroll
  for (int v = 0; v < 16; ++v) col[(size_t)(hi + 16 * v) << KB] = canon(x[v], p, pinv);
}

// pass B of every ModUp digit of one (lane, slot, chunk) + key inner product (see KmB)
__global__ void __launch_bounds__(256, 2) fwd_b_km(const KmB K) {
  extern __shared__ double dyn[];
  __shared__ u64 mbar;
  double* sm = dyn;                          // exchange rows
  double* stw = dyn + 16 * kStride;          // round-2 twiddle blob of (prime, chunk)
  double* acc1 = stw + kNttBlobTile;         // comp-1 accumulators: 16 private words per thread
  const u32 lane = blockIdx.x % K.nlanes, rest = blockIdx.x / K.nlanes;
  const u32 chunk = rest & 15, t = rest >> 4;
  const u32 e = t < K.level ? t : kSpecialBase + (t - K.level);
  const NttScale* sc = K.scale + e;
  const double p = sc->pd, pinv = sc->pinv;
  blob_init(&mbar);
  __syncthreads();
  blob_issue(&mbar, stw, K.tw[e].fb + (size_t)chunk * kNttBlobTile);
  pdl_wait();
  bool blob_ready = false;
  const u32 lo = threadIdx.x & 15, hi = threadIdx.x >> 4;
  const size_t s0 = (size_t)(chunk * 16 + hi) * 256 + 16 * lo;
  const size_t kcomp = (size_t)K.key_slots * K.n;
  const u32 ks = t < K.level ? t : K.chain + (t - K.level);
  const u64* kb = K.key + (size_t)ks * K.n + s0;
  double* sp = sm + hi * kStride;
  double acc0[16];
#pragma unroll
  for (int v = 0; v < 16; ++v) {
    acc0[v] = 0.0;
    acc1[v * 256 + threadIdx.x] = 0.0;
  }
  for (u32 j = 0; j < K.dnum; ++j) {
    const u32 lo_j = j * kAlpha, hi_j = lo_j + kAlpha < K.level ? lo_j + kAlpha : K.level;
    const bool own = t < K.level && t >= lo_j && t < hi_j;
    double y[16];
    if (own) {  // E_j(t) = d[t], already in the NTT domain
      const u64* dr = K.d + (size_t)lane * K.d_ls + (size_t)t * K.n + s0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        u64 a, b, c, dd;
        ld256(dr + 4 * k, a, b, c, dd);
        y[4 * k] = u2d(a);
        y[4 * k + 1] = u2d(b);
        y[4 * k + 2] = u2d(c);
        y[4 * k + 3] = u2d(dd);
      }
    } else {
      const u32 idx = j * K.nslots - lo_j + (t < lo_j ? t : t - (hi_j - lo_j));
      const u64* blk = K.ext + (size_t)lane * K.ext_ls + (size_t)idx * K.n + (size_t)(chunk * 16 + hi) * 256;
#pragma unroll
#if AEGIS_KM_EXT_CS
      for (int v = 0; v < 16; ++v) y[v] = dbits(__ldcs(blk + lo + 16 * v));
#else
      for (int v = 0; v < 16; ++v) y[v] = dbits(blk[lo + 16 * v]);
#endif
      double w[15];
#if AEGIS_BLOB_R1
      if (!blob_ready) {
        blob_wait(&mbar, 0);
        blob_ready = true;
      }
      load_w_blob1(w, stw + hi * kNttBlobSub);
#else
      load_w<0>(w, K.tw[e].fw, 256 + chunk * 16 + hi, 0);
#endif
      ct16(y, WArr{w}, p, pinv);
#pragma unroll
      for (int v = 0; v < 16; ++v) sp[lo + 17 * v] = y[v];
      __syncwarp();
      if (!blob_ready) {
        blob_wait(&mbar, 0);
        blob_ready = true;
      }
      load_w_blob(w, stw + hi * kNttBlobSub + lo);
#pragma unroll
      for (int v = 0; v < 16; ++v) y[v] = sp[17 * lo + v];
      __syncwarp();  // the rows are rewritten by the next digit
      ct16(y, WArr{w}, p, pinv);
    }
    const u64* k0 = kb + (size_t)j * 2 * kcomp;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      u64 a, b, c, dd;
#if AEGIS_KM_KEY_NA
      ld256na(k0 + 4 * k, a, b, c, dd);
#else
      ld256(k0 + 4 * k, a, b, c, dd);
#endif
      const double w0 = u2d(a), w1 = u2d(b), w2 = u2d(c), w3 = u2d(dd);
      acc0[4 * k] += mm(y[4 * k], w0, w0 * pinv, p);
      acc0[4 * k + 1] += mm(y[4 * k + 1], w1, w1 * pinv, p);
      acc0[4 * k + 2] += mm(y[4 * k + 2], w2, w2 * pinv, p);
      acc0[4 * k + 3] += mm(y[4 * k + 3], w3, w3 * pinv, p);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      u64 a, b, c, dd;
#if AEGIS_KM_KEY_NA
      ld256na(k0 + kcomp + 4 * k, a, b, c, dd);
#else
      ld256(k0 + kcomp + 4 * k, a, b, c, dd);
#endif
      const u64 kk[4] = {a, b, c, dd};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double wk = u2d(kk[i]);
        acc1[(4 * k + i) * 256 + threadIdx.x] += mm(y[4 * k + i], wk, wk * pinv, p);
      }
    }
  }
  if (!blob_ready) blob_wait(&mbar, 0);  // never leave the bulk copy in flight
  u64* a0 = K.acc + (size_t)lane * K.acc_ls + (size_t)t * K.n + s0;
  u64* a1 = a0 + (size_t)K.nslots * K.n;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    st256(a0 + 4 * k, canon(acc0[4 * k], p, pinv), canon(acc0[4 * k + 1], p, pinv), canon(acc0[4 * k + 2], p, pinv),
          canon(acc0[4 * k + 3], p, pinv));
    st256(a1 + 4 * k, canon(acc1[(4 * k) * 256 + threadIdx.x], p, pinv),
          canon(acc1[(4 * k + 1) * 256 + threadIdx.x], p, pinv), canon(acc1[(4 * k + 2) * 256 + threadIdx.x], p, pinv),
          canon(acc1[(4 * k + 3) * 256 + threadIdx.x], p, pinv));
  }
}
constexpr size_t kSmemKm = (size_t)(16 * kStride + kNttBlobTile + 4096) * sizeof(double);

constexpr size_t kSmemB = (size_t)(16 * kStride + kNttBlobTile) * sizeof(double);

// ---- one-launch-per-pass kernels (slot-major rows) ---------------------------
__device__ __forceinline__ RowRef slot_major(const NttLaunch& L, u32 row, u32& slot) {
  slot = row / L.nlanes;
  return row_ref(L, row - slot * L.nlanes, slot);
}
template <int KB = 8>
__global__ void __launch_bounds__(256, 3) fwd_a(const NttLaunch L) {
  __shared__ double sm[16 * kStride];
  u32 slot;
  pdl_wait();
  tile_fwd_a<KB>(L, slot_major(L, blockIdx.x >> (KB - 4), slot), blockIdx.x & ((1u << (KB - 4)) - 1), sm);
}
__global__ void __launch_bounds__(256, 3) fwd_b(const NttLaunch L) {
  extern __shared__ double dyn[];
  __shared__ u64 mbar;
  u32 slot;
  const RowRef rr = slot_major(L, blockIdx.x >> 4, slot);
  const u32 chunk = blockIdx.x & 15;
  blob_init(&mbar);
  __syncthreads();
  blob_issue(&mbar, dyn + 16 * kStride, L.tw[rr.prime].fb + (size_t)chunk * kNttBlobTile);
  pdl_wait();  // the twiddle blob is a constant table: its copy overlaps the predecessor's tail
  tile_fwd_b(L, rr, chunk, dyn, dyn + 16 * kStride, &mbar, 0);
}
#ifndef AEGIS_FIN_MINB
#define AEGIS_FIN_MINB 2
#endif
__global__ void __launch_bounds__(256, AEGIS_FIN_MINB) fwd_b_fin(const NttLaunch L, const NttFin F) {
  extern __shared__ double dyn[];
  __shared__ u64 mbar;
  const u32 row = blockIdx.x >> 4, chunk = blockIdx.x & 15;
  const u32 slot = row / L.nlanes, lane_v = row - slot * L.nlanes;
  blob_init(&mbar);
  __syncthreads();
  blob_issue(&mbar, dyn + 16 * kStride, L.tw[L.prime[slot]].fb + (size_t)chunk * kNttBlobTile);
  pdl_wait();
  tile_fwd_b_fin(L, F, lane_v, slot, chunk, dyn, dyn + 16 * kStride, &mbar, 0);
}
__global__ void __launch_bounds__(256, 3) inv_b(const NttLaunch L) {
  extern __shared__ double dyn[];
  __shared__ u64 mbar;
  u32 slot;
  const u32 row = blockIdx.x >> 4;
  const RowRef rr = slot_major(L, row, slot);
  const u32 chunk = blockIdx.x & 15;
  const u64* src = L.in_base ? L.in_base + (size_t)(row - slot * L.nlanes) * L.in_lane_stride +
                                   (size_t)L.in_slot_off[slot] * L.n
                             : rr.ptr;
  blob_init(&mbar);
  __syncthreads();
  blob_issue(&mbar, dyn + 16 * kStride, L.tw[rr.prime].ib + (size_t)chunk * kNttBlobTile);
  pdl_wait();
  tile_inv_b(L, rr, src, chunk, dyn, dyn + 16 * kStride, &mbar, 0);
}
template <int KB = 8>
__global__ void __launch_bounds__(256, 3) inv_a(const NttLaunch L) {
  __shared__ double sm[16 * kStride];
  u32 slot;
  pdl_wait();
  tile_inv_a<KB>(L, slot_major(L, blockIdx.x >> (KB - 4), slot), blockIdx.x & ((1u << (KB - 4)) - 1), sm);
}

// fused conversion + pass A, one launch per pass: tiles ordered (lane, chunk,
// slot fastest) so the CTAs converting one lane's column chunk run together
#ifndef AEGIS_CFWD_MINB
#define AEGIS_CFWD_MINB 3  // resident CTAs per SM the register cap is sized for
#endif
template <int K, int T>
__global__ void __launch_bounds__(256, AEGIS_CFWD_MINB) cfwd_a(const NttLaunch L, const NttConvIn C) {
  extern __shared__ double dyn[];  // exchange rows + (T-1) x 4096 parked targets
  pdl_wait();
  const u32 groups = (L.nslots + T - 1) / T;
  const u32 grp = blockIdx.x % groups, rest = blockIdx.x / groups;
  const u32 slot0 = grp * T, nt = L.nslots - slot0 < (u32)T ? L.nslots - slot0 : (u32)T;
  tile_cfwd_a<K, T>(L, C, rest >> 4, slot0, nt, rest & 15, dyn, reinterpret_cast<u64*>(dyn + 16 * kStride));
}

void init_attrs() {
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(fwd_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemB);
    cudaFuncSetAttribute(inv_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemB);
    cudaFuncSetAttribute(fwd_b_fin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemB);
    cudaFuncSetAttribute(fwd_b_km, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemKm);
    const int cs = (int)((16 * kStride) * sizeof(double) + (kConvTargets - 1) * 4096 * sizeof(u64));
    cudaFuncSetAttribute(cfwd_a<1, kConvTargets>, cudaFuncAttributeMaxDynamicSharedMemorySize, cs);
    cudaFuncSetAttribute(cfwd_a<2, kConvTargets>, cudaFuncAttributeMaxDynamicSharedMemorySize, cs);
    cudaFuncSetAttribute(cfwd_a<3, kConvTargets>, cudaFuncAttributeMaxDynamicSharedMemorySize, cs);
    cudaFuncSetAttribute(cfwd_a<4, kConvTargets>, cudaFuncAttributeMaxDynamicSharedMemorySize, cs);
    init = true;
  }
}

cudaError_t run(const NttLaunch& L, bool inverse, cudaStream_t st) {
  init_attrs();
  const u32 rows = L.nlanes * L.nslots;
  const dim3 grid(rows * 16), block(256);
  if (!inverse) {
    launch_pdl(fwd_a<8>, grid, block, 0, st, L);
    launch_pdl(fwd_b, grid, block, kSmemB, st, L);
  } else {
    launch_pdl(inv_b, grid, block, kSmemB, st, L);
    launch_pdl(inv_a<8>, grid, block, 0, st, L);
  }
  return cudaGetLastError();
}

// ---- N = 2^17 block pass: 512-point sub-transforms (global stages 8..16) ----
// A CTA owns 8 subs; warp w = sub w, lane = tau.  Rounds of 4, 4 and 1 stages
// (element patterns tau + 32v, (tau&1) + 2v + 32(tau>>1), 16 tau + v), two
// padded SMEM exchanges inside the warp.  Twiddles come from the w-only table:
// round 1 uniform per warp, round 2 per lane pair, round 3 eight contiguous
// words per lane (two 256-bit loads).  Input/output patterns are coalesced:
// loads `tau + 32v` (forward) / 256-bit rows (inverse), stores the reverse.
constexpr int kStride512 = 512 + 32 + 1;
__device__ __forceinline__ u32 pad16(u32 u) { return u + (u >> 4); }

__device__ __forceinline__ void load_w8(double (&w)[8], const double* tw, u32 t0, u32 tau) {
  const u64* q = reinterpret_cast<const u64*>(tw + ((size_t)t0 << 8) + 8 * tau);
  u64 a[8];
  ld256(q, a[0], a[1], a[2], a[3]);
  ld256(q + 4, a[4], a[5], a[6], a[7]);
#pragma unroll
  for (int k = 0; k < 8; ++k) w[k] = dbits(a[k]);
}

__global__ void __launch_bounds__(256, 3) fwd_b512(const NttLaunch L) {
  __shared__ double sm[8 * kStride512];
  u32 slot;
  const RowRef rr = slot_major(L, blockIdx.x >> 5, slot);
  const u32 chunk = blockIdx.x & 31;
  const NttScale* sc = L.scale + rr.prime;
  const double p = sc->pd, pinv = sc->pinv;
  const double* tw = L.tw[rr.prime].fw;
  const u32 tau = threadIdx.x & 31, sub = threadIdx.x >> 5;
  const u32 t0 = 256 + chunk * 8 + sub, tl = tau & 1, th = tau >> 1;
  u64* blk = rr.ptr + (size_t)(chunk * 8 + sub) * 512;
  double x[16], w[15];
#pragma unroll
  for (int v = 0; v < 16; ++v) x[v] = dbits(blk[tau + 32 * v]);
  load_w<0>(w, tw, t0, 0);
  ct16(x, WArr{w}, p, pinv);
  double* sp = sm + sub * kStride512;
#pragma unroll
  for (int v = 0; v < 16; ++v) sp[pad16(tau + 32 * v)] = x[v];
  __syncwarp();
  load_w<4>(w, tw, t0, th);
#pragma unroll
  for (int v = 0; v < 16; ++v) x[v] = sp[pad16(tl + 2 * v + 32 * th)];
  ct16(x, WArr{w}, p, pinv);
  __syncwarp();
#pragma unroll
  for (int v = 0; v < 16; ++v) sp[pad16(tl + 2 * v + 32 * th)] = x[v];
  __syncwarp();
  double w8[8];
  load_w8(w8, tw, t0, tau);
#pragma unroll
  for (int v = 0; v < 16; ++v) x[v] = sp[pad16(16 * tau + v)];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double t = mm(x[2 * k + 1], w8[k], w8[k] * pinv, p);
    const double a = x[2 * k];
    x[2 * k] = a + t;
    x[2 * k + 1] = a - t;
  }
  u64* o = blk + 16 * tau;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    st256(o + 4 * k, canon(x[4 * k], p, pinv), canon(x[4 * k + 1], p, pinv), canon(x[4 * k + 2], p, pinv),
          canon(x[4 * k + 3], p, pinv));
}

__global__ void __launch_bounds__(256, 3) inv_b512(const NttLaunch L) {
  __shared__ double sm[8 * kStride512];
  u32 slot;
  const RowRef rr = slot_major(L, blockIdx.x >> 5, slot);
  const u32 chunk = blockIdx.x & 31;
  const NttScale* sc = L.scale + rr.prime;
  const double p = sc->pd, pinv = sc->pinv;
  const double* tw = L.tw[rr.prime].iw;
  const u32 tau = threadIdx.x & 31, sub = threadIdx.x >> 5;
  const u32 t0 = 256 + chunk * 8 + sub, tl = tau & 1, th = tau >> 1;
  u64* blk = rr.ptr + (size_t)(chunk * 8 + sub) * 512;
  double x[16], w[15];
  {
    u64 raw[16];
#pragma unroll
    for (int k = 0; k < 4; ++k) ld256(blk + 16 * tau + 4 * k, raw[4 * k], raw[4 * k + 1], raw[4 * k + 2], raw[4 * k + 3]);
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = u2d(raw[v]);
  }
  double w8[8];
  load_w8(w8, tw, t0, tau);
#pragma unroll
  for (int k = 0; k < 8; ++k) {  // GS stage 8
    const double a = x[2 * k], b = x[2 * k + 1];
    x[2 * k] = a + b;
    x[2 * k + 1] = mm(a - b, w8[k], w8[k] * pinv, p);
  }
  double* sp = sm + sub * kStride512;
#pragma unroll
  for (int v = 0; v < 16; ++v) sp[pad16(16 * tau + v)] = red(x[v], p, pinv);
  __syncwarp();
  load_w<4>(w, tw, t0, th);
#pragma unroll
  for (int v = 0; v < 16; ++v) x[v] = sp[pad16(tl + 2 * v + 32 * th)];
  gs16<false>(x, WArr{w}, p, pinv, sc);
  __syncwarp();
#pragma unroll
  for (int v = 0; v < 16; ++v) sp[pad16(tl + 2 * v + 32 * th)] = red(x[v], p, pinv);
  __syncwarp();
  load_w<0>(w, tw, t0, 0);
#pragma unroll
  for (int v = 0; v < 16; ++v) x[v] = sp[pad16(tau + 32 * v)];
  gs16<false>(x, WArr{w}, p, pinv, sc);
#pragma unroll
  for (int v = 0; v < 16; ++v) blk[tau + 32 * v] = bitsd(red(x[v], p, pinv));
}

// N = 2^17 = 256 x 512: column pass (256-point sub-transforms on 512 columns)
// + the 512-point block pass above.
cudaError_t run17(const NttLaunch& L, bool inverse, cudaStream_t st) {
  init_attrs();
  const u32 rows = L.nlanes * L.nslots;
  const dim3 grid(rows * 32), block(256);
  if (!inverse) {
    fwd_a<9><<<grid, block, 0, st>>>(L);
    fwd_b512<<<grid, block, 0, st>>>(L);
  } else {
    inv_b512<<<grid, block, 0, st>>>(L);
    inv_a<9><<<grid, block, 0, st>>>(L);
  }
  return cudaGetLastError();
}

// kernel probe brackets (see KernelProbe)
inline void probe_mark(int kind, cudaStream_t st) {
  if (!g_probe || g_probe->kind != kind) return;
  cudaEvent_t e;
  if (cudaEventCreate(&e) != cudaSuccess) return;
  cudaEventRecord(e, st);
  g_probe->ev.push_back(e);
}
inline void probe_done(int kind, cudaStream_t st, double bytes) {
  if (!g_probe || g_probe->kind != kind) return;
  probe_mark(kind, st);
  g_probe->alg_bytes += bytes;
  ++g_probe->launches;
}

cudaError_t run_km(const KmB& K, cudaStream_t st) {
  init_attrs();
  probe_mark(kProbeFwdBKm, st);
  launch_pdl(fwd_b_km, dim3(K.nlanes * 16 * K.nslots), dim3(256), kSmemKm, st, K);
  // per (lane, slot): dnum digit limbs in, 2 accumulators out; the keys once per launch
  probe_done(kProbeFwdBKm, st,
             8.0 * K.n * ((double)K.nlanes * K.nslots * (K.dnum + 2) + 2.0 * K.dnum * K.nslots));
  return cudaGetLastError();
}

cudaError_t run_conv(const NttLaunch& L, const NttConvIn& C, const NttFin* fin, cudaStream_t st, bool pass_a_only) {
  init_attrs();
  const dim3 grid(L.nlanes * L.nslots * 16), block(256);
  constexpr int T = kConvTargets;
  const size_t smem = (size_t)(16 * kStride) * sizeof(double) + (size_t)(T - 1) * 4096 * sizeof(u64);
  const dim3 cgrid(L.nlanes * 16 * ((L.nslots + T - 1) / T));
  probe_mark(kProbeCfwdA, st);
  switch (C.k) {
    case 1: launch_pdl(cfwd_a<1, T>, cgrid, block, smem, st, L, C); break;
    case 2: launch_pdl(cfwd_a<2, T>, cgrid, block, smem, st, L, C); break;
    case 3: launch_pdl(cfwd_a<3, T>, cgrid, block, smem, st, L, C); break;
    case 4: launch_pdl(cfwd_a<4, T>, cgrid, block, smem, st, L, C); break;
    default: return cudaErrorInvalidValue;
  }
  // k prepared source limbs + the overflow-count row read once per lane, every target limb written once
  probe_done(kProbeCfwdA, st, 8.0 * L.n * (double)L.nlanes * (L.nslots + C.k + 1));
  if (pass_a_only) return cudaGetLastError();
  if (fin) {
    probe_mark(kProbeFwdBFin, st);
    launch_pdl(fwd_b_fin, grid, block, kSmemB, st, L, *fin);
    // per (virtual lane, slot): pass-A intermediate + x (+ add) in, out written
    const double adds = fin->add ? (double)L.nlanes * std::min(fin->add_comps, fin->comps) / fin->comps : 0.0;
    probe_done(kProbeFwdBFin, st, 8.0 * L.n * (double)L.nslots * (3.0 * L.nlanes + adds));
  } else {
    launch_pdl(fwd_b, grid, block, kSmemB, st, L);
  }
  return cudaGetLastError();
}

cudaError_t run_fin(const NttLaunch& L, const NttFin& fin, cudaStream_t st) {
  init_attrs();
  const dim3 grid(L.nlanes * L.nslots * 16), block(256);
  launch_pdl(fwd_a<8>, grid, block, 0, st, L);
  probe_mark(kProbeFwdBFin, st);
  launch_pdl(fwd_b_fin, grid, block, kSmemB, st, L, fin);
  const double adds = fin.add ? (double)L.nlanes * std::min(fin.add_comps, fin.comps) / fin.comps : 0.0;
  probe_done(kProbeFwdBFin, st, 8.0 * L.n * (double)L.nslots * (3.0 * L.nlanes + adds));
  return cudaGetLastError();
}

}  // namespace v2

template <int IMPL>
cudaError_t run_impl(const NttLaunch& L, int log_n, bool inverse, cudaStream_t st) {
  const u32 rows = L.nlanes * L.nslots;
  const int kA = log_n / 2, kB = log_n - kA;
  cudaError_t e;
  if (!inverse) {
    e = dispatch_pass<0, false, IMPL>(kA, L, kA, kB, rows, 0, st);
    if (e != cudaSuccess) return e;
    return dispatch_pass<1, false, IMPL>(kB, L, kA, kB, rows, 0, st);
  }
  e = dispatch_pass<1, true, IMPL>(kB, L, kA, kB, rows, 0, st);
  if (e != cudaSuccess) return e;
  return dispatch_pass<0, true, IMPL>(kA, L, kA, kB, rows, 1, st);
}

}  // namespace

void ntt_build_blob(const double* tab, double* blob) {
  for (int c = 0; c < 16; ++c)
    for (int b = 0; b < 16; ++b) {
      double* d = blob + (size_t)c * kNttBlobTile + (size_t)b * kNttBlobSub;
      const unsigned t0 = 256 + 16 * c + b;
      for (int sg = 0; sg < 4; ++sg)
        for (int q = 0; q < (1 << sg); ++q) {
          for (int tau = 0; tau < 16; ++tau) d[v2::tw2_off(sg, q) + tau] = tab[(t0 << (4 + sg)) + (tau << sg) + q];
          d[v2::tw2_off(sg, q) + 16] = 0.0;
          d[v2::kTw1 + (1 << sg) - 1 + q] = tab[(t0 << sg) + q];
        }
    }
}

cudaError_t ntt_conv_fwd(const NttLaunch& L, const NttConvIn& c, const NttFin* fin, cudaStream_t st,
                         bool pass_a_only) {
  if (L.nlanes * L.nslots == 0) return cudaSuccess;
  return v2::run_conv(L, c, fin, st, pass_a_only);
}
cudaError_t ntt_fwd_b_keymul(const KmB& k, cudaStream_t st) {
  if (!k.nlanes || !k.nslots) return cudaSuccess;
  return v2::run_km(k, st);
}
cudaError_t ntt_fwd_fin(const NttLaunch& L, const NttFin& fin, cudaStream_t st) {
  if (L.nlanes * L.nslots == 0) return cudaSuccess;
  return v2::run_fin(L, fin, st);
}

KernelProbe* g_probe = nullptr;

bool ntt_v2_active(int log_n) { return log_n == 16 && g_ntt_impl == kNttF64 && g_ntt_v2; }

cudaError_t ntt_run(const NttLaunch& L, int log_n, bool inverse, cudaStream_t st) {
  if (L.nlanes * L.nslots == 0) return cudaSuccess;
  if (L.in_base && !(inverse && ntt_v2_active(log_n))) return cudaErrorInvalidValue;
  if (log_n == 16 && g_ntt_impl == kNttF64 && g_ntt_v2) return v2::run(L, inverse, st);
  if (log_n == 17 && g_ntt_impl == kNttF64 && g_ntt_v2 && !L.in_base) return v2::run17(L, inverse, st);
  return g_ntt_impl == kNttF64 ? run_impl<kNttF64>(L, log_n, inverse, st) : run_impl<kNttInt>(L, log_n, inverse, st);
}

}  // namespace aegis

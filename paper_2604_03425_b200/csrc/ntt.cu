// ntt.cu -- batched negacyclic NTT / INTT for sm_100a.
//
// Semantics: exactly NegacyclicNtt::forward / ::inverse of rns_math.hpp:68-100
// (Cooley-Tukey DIT, natural order in -> bit-reversed evaluation order out;
// Gentleman-Sande inverse followed by the N^{-1} scale, which we fold into the
// last GS stage).  psi and the bit-reversed twiddle tables are the
// reference's (rns_math.hpp:53-61, 103-117), built on the host in context.cu.
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
// Twiddles are (w, floor(w 2^64/p)) pairs read as one 128-bit load.
#include "ntt.h"

namespace aegis {

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

// Lazy reduction (Harvey): p < 2^48 leaves 16 bits of headroom in a u64, so
// butterflies never reduce.  CT: X' = X + T, Y' = X + 2p - T with
// T = Shoup(Y) in [0, 2p): bounds grow by 2p per stage (< 35p after 17 stages).
// GS: X' = X + Y, Y' = Shoup(X + B - Y) with B = 2^d p the bound after d
// stages: the sum path doubles per stage, so the inverse reduces once between
// its two passes.  Only pass outputs leaving the NTT are made canonical.
__device__ __forceinline__ u64 reduce_lazy(u64 x, u64 p, u64 mu) {
  const u64 r = x - __umul64hi(x, mu) * p;  // in [0, 2p)
  return r >= p ? r - p : r;
}

// One radix-2^R round of forward CT stages s0 .. s0+R-1 on the sub-problem at sp.
template <int LOGM>
__device__ __forceinline__ void ct_round(u64* sp, u32 tau, int s0, u32 t0,
                                         const ulonglong2* __restrict__ tw, u64 p) {
  using C = SubCfg<LOGM>;
  constexpr int R = C::R;
  const int lo_bits = LOGM - s0 - R;
  const u32 tau_lo = tau & ((1u << lo_bits) - 1);
  const u32 tau_hi = tau >> lo_bits;
  const u32 base = tau_lo | (tau_hi << (lo_bits + R));
  const u64 two_p = 2 * p;
  u64 x[1 << R];
#pragma unroll
  for (int v = 0; v < (1 << R); ++v) x[v] = sp[pad_idx(base | ((u32)v << lo_bits))];
#pragma unroll
  for (int sg = 0; sg < R; ++sg) {
    const int s = s0 + sg;
    const int half = 1 << (R - sg - 1);
#pragma unroll
    for (int v = 0; v < (1 << R); ++v) {
      if (v & half) continue;
      const u32 i = (tau_hi << sg) | ((u32)v >> (R - sg));
      const ulonglong2 w = tw[(t0 << s) + i];
      const u64 a = x[v];
      const u64 t = shoup_lazy(x[v + half], w.x, w.y, p);
      x[v] = a + t;
      x[v + half] = a + two_p - t;
    }
  }
#pragma unroll
  for (int v = 0; v < (1 << R); ++v) sp[pad_idx(base | ((u32)v << lo_bits))] = x[v];
}

// One radix-2^R round of inverse GS stages s0+R-1 .. s0 (descending).  `depth`
// counts GS stages already applied since values were last canonical.  When
// `last` is set the round contains the global final stage (s == 0 of pass A):
// there N^{-1} is folded into both outputs, which come out canonical.
template <int LOGM>
__device__ __forceinline__ void gs_round(u64* sp, u32 tau, int s0, u32 t0,
                                         const ulonglong2* __restrict__ tw, u64 p, int depth,
                                         bool last, const NttScale& sc) {
  using C = SubCfg<LOGM>;
  constexpr int R = C::R;
  const int lo_bits = LOGM - s0 - R;
  const u32 tau_lo = tau & ((1u << lo_bits) - 1);
  const u32 tau_hi = tau >> lo_bits;
  const u32 base = tau_lo | (tau_hi << (lo_bits + R));
  u64 x[1 << R];
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
      const u32 i = (tau_hi << sg) | ((u32)v >> (R - sg));
      const u64 a = x[v], b = x[v + half];
      if (scale) {
        // s == 0: single twiddle inv[1]; fold N^{-1} into both outputs
        x[v] = shoup(a + b, sc.n_inv, sc.n_inv_p, p);
        x[v + half] = shoup(a + bound - b, sc.w1n, sc.w1n_p, p);
      } else {
        const ulonglong2 w = tw[(t0 << s) + i];
        x[v] = a + b;
        x[v + half] = shoup_lazy(a + bound - b, w.x, w.y, p);
      }
    }
  }
#pragma unroll
  for (int v = 0; v < (1 << R); ++v) sp[pad_idx(base | ((u32)v << lo_bits))] = x[v];
}

// MODE 0: columns (pass A), MODE 1: contiguous blocks (pass B).
//   forward : pass A (canonical -> lazy), pass B (lazy -> canonical)
//   inverse : pass B (canonical -> lazy < 2^kB p), pass A (reduce on load -> canonical)
template <int LOGM, int MODE, bool INV>
__global__ void __launch_bounds__(256) ntt_pass_kernel(const NttLaunch L, int kA, int kB,
                                                       int subs_per_cta, int scale_last) {
  using C = SubCfg<LOGM>;
  extern __shared__ u64 smem[];
  const u32 ctas_per_row = MODE == 0 ? (1u << kB) / subs_per_cta : (1u << kA) / subs_per_cta;
  const u32 row = blockIdx.x / ctas_per_row;
  const u32 chunk = blockIdx.x - row * ctas_per_row;
  const RowInfo ri = row_info(L, row);
  const PrimeTw pt = L.tw[ri.prime];
  const NttScale sc = L.scale[ri.prime];
  const ulonglong2* __restrict__ tw = INV ? pt.inv : pt.fwd;
  const u64 p = pt.p;
  const u32 nthreads = blockDim.x;
  const u32 total = subs_per_cta * C::M;
  const bool reduce_in = INV && MODE == 0;    // lazy intermediate of the inverse
  const bool reduce_out = !INV && MODE == 1;  // end of the forward transform

  // ---- load (coalesced) ----
  if (MODE == 0) {
    const u32 c0 = chunk * subs_per_cta;
    const u32 cmask = subs_per_cta - 1;
    const int clog = __ffs(subs_per_cta) - 1;
    for (u32 e = threadIdx.x; e < total; e += nthreads) {
      const u32 c = e & cmask, u = e >> clog;
      u64 v = ri.ptr[c0 + c + ((size_t)u << kB)];
      if (reduce_in) v = reduce_lazy(v, p, sc.mu64);
      smem[c * C::STRIDE + pad_idx(u)] = v;
    }
  } else {
    const size_t off = (size_t)chunk * total;
    for (u32 e = threadIdx.x; e < total; e += nthreads) {
      const u32 b = e >> LOGM, v = e & (C::M - 1);
      smem[b * C::STRIDE + pad_idx(v)] = ri.ptr[off + e];
    }
  }
  __syncthreads();

  const u32 sub = threadIdx.x / C::TPS;
  const u32 tau = threadIdx.x - sub * C::TPS;
  u64* sp = smem + sub * C::STRIDE;
  const u32 t0 = MODE == 0 ? 1u : (1u << kA) + chunk * subs_per_cta + sub;
  // block = subs_per_cta * TPS threads exactly, so every thread owns work
  if (!INV) {
#pragma unroll
    for (int rd = 0; rd < C::ROUNDS; ++rd) {
      ct_round<LOGM>(sp, tau, rd * C::R, t0, tw, p);
      if (rd + 1 < C::ROUNDS) {
        if (C::TPS > 32) __syncthreads(); else __syncwarp();
      }
    }
  } else {
#pragma unroll
    for (int rd = C::ROUNDS - 1; rd >= 0; --rd) {
      gs_round<LOGM>(sp, tau, rd * C::R, t0, tw, p, (C::ROUNDS - 1 - rd) * C::R, scale_last && rd == 0, sc);
      if (rd > 0) {
        if (C::TPS > 32) __syncthreads(); else __syncwarp();
      }
    }
  }
  __syncthreads();

  // ---- store (coalesced) ----
  if (MODE == 0) {
    const u32 c0 = chunk * subs_per_cta;
    const u32 cmask = subs_per_cta - 1;
    const int clog = __ffs(subs_per_cta) - 1;
    for (u32 e = threadIdx.x; e < total; e += nthreads) {
      const u32 c = e & cmask, u = e >> clog;
      ri.ptr[c0 + c + ((size_t)u << kB)] = smem[c * C::STRIDE + pad_idx(u)];
    }
  } else {
    const size_t off = (size_t)chunk * total;
    for (u32 e = threadIdx.x; e < total; e += nthreads) {
      const u32 b = e >> LOGM, v = e & (C::M - 1);
      u64 x = smem[b * C::STRIDE + pad_idx(v)];
      if (reduce_out) x = reduce_lazy(x, p, sc.mu64);
      ri.ptr[off + e] = x;
    }
  }
}

template <int LOGM, int MODE, bool INV>
cudaError_t launch_pass(const NttLaunch& L, int kA, int kB, u32 rows, int scale_last,
                        cudaStream_t st) {
  using C = SubCfg<LOGM>;
  const int nsub_total = MODE == 0 ? (1 << kB) : (1 << kA);
  int subs = 256 / C::TPS;
  if (subs > nsub_total) subs = nsub_total;
  if (subs < 1) subs = 1;
  const u32 ctas_per_row = nsub_total / subs;
  const size_t smem = (size_t)subs * C::STRIDE * sizeof(u64);
  auto kern = ntt_pass_kernel<LOGM, MODE, INV>;
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  const dim3 grid(rows * ctas_per_row);
  const dim3 block(subs * C::TPS);
  kern<<<grid, block, smem, st>>>(L, kA, kB, subs, scale_last);
  return cudaGetLastError();
}

template <int MODE, bool INV>
cudaError_t dispatch_pass(int logm, const NttLaunch& L, int kA, int kB, u32 rows, int scale_last,
                          cudaStream_t st) {
  switch (logm) {
    case 1: return launch_pass<1, MODE, INV>(L, kA, kB, rows, scale_last, st);
    case 2: return launch_pass<2, MODE, INV>(L, kA, kB, rows, scale_last, st);
    case 3: return launch_pass<3, MODE, INV>(L, kA, kB, rows, scale_last, st);
    case 4: return launch_pass<4, MODE, INV>(L, kA, kB, rows, scale_last, st);
    case 5: return launch_pass<5, MODE, INV>(L, kA, kB, rows, scale_last, st);
    case 6: return launch_pass<6, MODE, INV>(L, kA, kB, rows, scale_last, st);
    case 7: return launch_pass<7, MODE, INV>(L, kA, kB, rows, scale_last, st);
    case 8: return launch_pass<8, MODE, INV>(L, kA, kB, rows, scale_last, st);
    case 9: return launch_pass<9, MODE, INV>(L, kA, kB, rows, scale_last, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

cudaError_t ntt_run(const NttLaunch& L, int log_n, bool inverse, cudaStream_t st) {
  const u32 rows = L.nlanes * L.nslots;
  if (rows == 0) return cudaSuccess;
  const int kA = log_n / 2, kB = log_n - kA;
  cudaError_t e;
  if (!inverse) {
    e = dispatch_pass<0, false>(kA, L, kA, kB, rows, 0, st);
    if (e != cudaSuccess) return e;
    return dispatch_pass<1, false>(kB, L, kA, kB, rows, 0, st);
  }
  e = dispatch_pass<1, true>(kB, L, kA, kB, rows, 0, st);
  if (e != cudaSuccess) return e;
  return dispatch_pass<0, true>(kA, L, kA, kB, rows, 1, st);
}

}  // namespace aegis

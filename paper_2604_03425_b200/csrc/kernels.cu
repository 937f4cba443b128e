// kernels.cu -- elementwise, basis-conversion, key-product and PCMM kernels.
//
// All of these are HBM-streaming kernels over [lane][comp][limb][N] u64
// bundles: a CTA owns a contiguous chunk of one limb row, so
// every warp access is a 256-byte (or 512-byte with ulonglong2) coalesced
// segment; per-row constants (prime, lane mapping) are computed once per CTA.
#include "kernels.h"

namespace aegis {

namespace {

constexpr int kThreads = 256;
constexpr int kPerThread = 2;
constexpr u32 kChunk = kThreads * kPerThread;  // coefficients per CTA

inline u32 chunks_of(u32 n) { return n >= kChunk ? n / kChunk : 1; }

// ---------------------------------------------------------------------------
// PRNG fills
// ---------------------------------------------------------------------------
__global__ void fill_uniform_kernel(View v, u32 comps, u32 limbs, u32 n, u64 seed, u64 tag, u64 a,
                                    const u32* __restrict__ limb_ext, const PrimeConst* __restrict__ pc,
                                    u32 cpr) {
  const u32 row = blockIdx.x / cpr, chunk = blockIdx.x - row * cpr;
  const u32 lb = row % limbs, rest = row / limbs, comp = rest % comps, lane = rest / comps;
  const u32 e = limb_ext[lb];
  const PrimeConst P = pc[e];
  const u64 rk = row_key(seed, tag, a, lane, comp, lb);
  u64* dst = v.limb(lane, comp, lb, n);
  for (u32 x = chunk * kChunk + threadIdx.x; x < n && x < (chunk + 1) * kChunk; x += kThreads)
    dst[x] = uniform_at(rk, x, P.p, P.shift);
}

__global__ void fill_key_kernel(u64* key, u32 slots, u32 n, u64 seed, u64 key_id,
                                const u32* __restrict__ slot_ext, const PrimeConst* __restrict__ pc,
                                u32 cpr) {
  const u32 row = blockIdx.x / cpr, chunk = blockIdx.x - row * cpr;
  const u32 slot = row % slots, rest = row / slots, comp = rest % 2, digit = rest / 2;
  const u32 e = slot_ext[slot];
  const PrimeConst P = pc[e];
  // tag 3: (key_id, digit, comp, ext prime) -- matches oracle key_limb()
  const u64 rk = row_key(seed, 3, key_id, digit, comp, e);
  u64* dst = key + (size_t)row * n;
  for (u32 x = chunk * kChunk + threadIdx.x; x < n && x < (chunk + 1) * kChunk; x += kThreads)
    dst[x] = uniform_at(rk, x, P.p, P.shift);
}

// ---------------------------------------------------------------------------
// Eval-domain automorphism: NTT(auto_k a)[j] = A[brv(((2 brv(j) + 1) k mod 2N - 1) / 2)]
// ---------------------------------------------------------------------------
__global__ void automorphism_kernel(View out, LaneMap om, View in, LaneMap im, u32 nlanes, u32 comps,
                                    u32 limbs, u32 log_n, u64 galois, u32 cpr) {
  const u32 n = 1u << log_n;
  const u32 row = blockIdx.x / cpr, chunk = blockIdx.x - row * cpr;
  const u32 lb = row % limbs, rest = row / limbs, comp = rest % comps, l = rest / comps;
  const u64* src = in.limb(im.at(l, nlanes), comp, lb, n);
  u64* dst = out.limb(om.at(l, nlanes), comp, lb, n);
  const u32 mask = 2 * n - 1;
  const u32 k = (u32)(galois & mask);
  for (u32 j = chunk * kChunk + threadIdx.x; j < n && j < (chunk + 1) * kChunk; j += kThreads) {
    const u32 bj = __brev(j) >> (32 - log_n);
    const u32 e = ((2 * bj + 1) * k) & mask;
    dst[j] = __ldg(src + (__brev((e - 1) >> 1) >> (32 - log_n)));
  }
}

// ---------------------------------------------------------------------------
// CMult tensor product and CAdd
// ---------------------------------------------------------------------------
__global__ void cmult_kernel(View out, u32 out_lane0, View a, LaneMap ma, View b, LaneMap mb,
                             u32 nlanes, u32 limbs, u32 n, const PrimeConst* __restrict__ pc, u32 cpr) {
  const u32 row = blockIdx.x / cpr, chunk = blockIdx.x - row * cpr;
  const u32 lb = row % limbs, l = row / limbs;
  const PrimeConst P = pc[lb];
  const u32 la = ma.at(l, nlanes), lbn = mb.at(l, nlanes);
  const u64* a0 = a.limb(la, 0, lb, n);
  const u64* a1 = a.limb(la, 1, lb, n);
  const u64* b0 = b.limb(lbn, 0, lb, n);
  const u64* b1 = b.limb(lbn, 1, lb, n);
  u64* d0 = out.limb(out_lane0 + l, 0, lb, n);
  u64* d1 = out.limb(out_lane0 + l, 1, lb, n);
  u64* d2 = out.limb(out_lane0 + l, 2, lb, n);
  for (u32 x = chunk * kChunk + threadIdx.x; x < n && x < (chunk + 1) * kChunk; x += kThreads) {
    const u64 x0 = a0[x], x1 = a1[x], y0 = b0[x], y1 = b1[x];
    d0[x] = mul_mod(x0, y0, P.p, P.mu104);
    u128 s = mul_wide(x0, y1);
    mac(s, x1, y0);
    d1[x] = reduce104(s, P.p, P.mu104);
    d2[x] = mul_mod(x1, y1, P.p, P.mu104);
  }
}

// 4 contiguous coefficients per thread, 256-bit accesses, streaming stores
// (the tensor product is HBM-bound: 7 limb streams per limb).  n % 1024 == 0.
__global__ void __launch_bounds__(256) cmult4_kernel(View out, u32 out_lane0, View a, LaneMap ma, View b, LaneMap mb,
                                                     u32 nlanes, u32 limbs, u32 n, const PrimeConst* __restrict__ pc) {
  const u32 cpr = n / 1024;
  const u32 row = blockIdx.x / cpr, chunk = blockIdx.x - row * cpr;
  const u32 lb = row % limbs, l = row / limbs;
  const PrimeConst P = pc[lb];
  const u32 la = ma.at(l, nlanes), lbn = mb.at(l, nlanes);
  const u32 x = (chunk * 256 + threadIdx.x) * 4;
  u64 a0[4], a1[4], b0[4], b1[4];
  ld256g(a.limb(la, 0, lb, n) + x, a0[0], a0[1], a0[2], a0[3]);  // operands may be wrapped: keep them cacheable
  ld256g(a.limb(la, 1, lb, n) + x, a1[0], a1[1], a1[2], a1[3]);
  ld256g(b.limb(lbn, 0, lb, n) + x, b0[0], b0[1], b0[2], b0[3]);
  ld256g(b.limb(lbn, 1, lb, n) + x, b1[0], b1[1], b1[2], b1[3]);
  u64 d0[4], d1[4], d2[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    d0[i] = mul_mod(a0[i], b0[i], P.p, P.mu104);
    u128 s = mul_wide(a0[i], b1[i]);
    mac(s, a1[i], b0[i]);
    d1[i] = reduce104(s, P.p, P.mu104);
    d2[i] = mul_mod(a1[i], b1[i], P.p, P.mu104);
  }
  st256cs(out.limb(out_lane0 + l, 0, lb, n) + x, d0[0], d0[1], d0[2], d0[3]);
  st256cs(out.limb(out_lane0 + l, 1, lb, n) + x, d1[0], d1[1], d1[2], d1[3]);
  st256cs(out.limb(out_lane0 + l, 2, lb, n) + x, d2[0], d2[1], d2[2], d2[3]);
}

// CMult of a ciphertext with itself (the softmax / GELU / LayerNorm squaring
// chains, he_ir.hpp:305-322): (a0^2, 2 a0 a1, a1^2) -- 2 operand streams
// instead of 4 (5 limb streams per limb instead of 7), 3 products instead of 4.
__global__ void __launch_bounds__(256) square4_kernel(View out, u32 out_lane0, View a, LaneMap ma, u32 nlanes,
                                                      u32 limbs, u32 n, const PrimeConst* __restrict__ pc) {
  const u32 cpr = n / 1024;
  const u32 row = blockIdx.x / cpr, chunk = blockIdx.x - row * cpr;
  const u32 lb = row % limbs, l = row / limbs;
  const PrimeConst P = pc[lb];
  const u32 la = ma.at(l, nlanes);
  const u32 x = (chunk * 256 + threadIdx.x) * 4;
  u64 a0[4], a1[4];
  ld256g(a.limb(la, 0, lb, n) + x, a0[0], a0[1], a0[2], a0[3]);
  ld256g(a.limb(la, 1, lb, n) + x, a1[0], a1[1], a1[2], a1[3]);
  u64 d0[4], d1[4], d2[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    d0[i] = mul_mod(a0[i], a0[i], P.p, P.mu104);
    u128 s = mul_wide(a0[i], a1[i]);
    mac(s, a1[i], a0[i]);
    d1[i] = reduce104(s, P.p, P.mu104);
    d2[i] = mul_mod(a1[i], a1[i], P.p, P.mu104);
  }
  st256cs(out.limb(out_lane0 + l, 0, lb, n) + x, d0[0], d0[1], d0[2], d0[3]);
  st256cs(out.limb(out_lane0 + l, 1, lb, n) + x, d1[0], d1[1], d1[2], d1[3]);
  st256cs(out.limb(out_lane0 + l, 2, lb, n) + x, d2[0], d2[1], d2[2], d2[3]);
}

// 8 contiguous coefficients per thread with 256-bit accesses (HBM-bound).
// The accumulator / first operand streams (evict-first) so a wrapped second
// operand (e.g. the 48 product lanes added into 1,536 score lanes) stays in L2.
__global__ void __launch_bounds__(256) cadd_kernel(View out, u32 out_lane0, View a, LaneMap ma, View b, LaneMap mb,
                                                   int acc, u32 nlanes, u32 comps, u32 limbs, u32 n,
                                                   const PrimeConst* __restrict__ pc, u32 cpr) {
  const u32 row = blockIdx.x / cpr, chunk = blockIdx.x - row * cpr;
  const u32 lb = row % limbs, rest = row / limbs, comp = rest % comps, l = rest / comps;
  const u64 p = pc[lb].p;
  const u64* x = a.limb(ma.at(l, nlanes), comp, lb, n);
  u64* d = out.limb(out_lane0 + l, comp, lb, n);
  const u64* y = acc ? d : b.limb(mb.at(l, nlanes), comp, lb, n);
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const u32 t = (chunk * 512 + k * 256 + threadIdx.x) * 4;
    if (t >= n) return;
    u64 x0, x1, x2, x3, y0, y1, y2, y3;
    if (acc) {  // d += x: d streams, x (possibly wrapped) is kept in L2
      ld256g(x + t, x0, x1, x2, x3);
      ld256cs(y + t, y0, y1, y2, y3);
    } else {
      ld256cs(x + t, x0, x1, x2, x3);
      ld256g(y + t, y0, y1, y2, y3);
    }
    st256cs(d + t, add_mod(x0, y0, p), add_mod(x1, y1, p), add_mod(x2, y2, p), add_mod(x3, y3, p));
  }
}

__global__ void copy_kernel(View dst, u32 dst_lane0, View src, LaneMap sm, u32 nlanes, u32 comps,
                            u32 limbs, u32 src_limb0, u32 n, u32 cpr) {
  const u32 row = blockIdx.x / cpr, chunk = blockIdx.x - row * cpr;
  const u32 lb = row % limbs, rest = row / limbs, comp = rest % comps, l = rest / comps;
  const u64* s = src.limb(sm.at(l, nlanes), comp, src_limb0 + lb, n);
  u64* d = dst.limb(dst_lane0 + l, comp, lb, n);
  for (u32 t = chunk * kChunk + threadIdx.x; t < n && t < (chunk + 1) * kChunk; t += kThreads) d[t] = s[t];
}

__global__ void hash_kernel(View v, u32 lane0, u32 comps, u32 limbs, u32 n, unsigned long long* out, u32 cpr) {
  const u32 row = blockIdx.x / cpr, chunk = blockIdx.x - row * cpr;
  const u32 lb = row % limbs, rest = row / limbs, comp = rest % comps, lane = lane0 + rest / comps;
  const u64* s = v.limb(lane, comp, lb, n);
  const u64 base = ((u64)lane * comps * limbs + (u64)comp * limbs + lb) * n;  // dense position
  u64 h = 0;
  for (u32 t = chunk * kChunk + threadIdx.x; t < n && t < (chunk + 1) * kChunk; t += kThreads)
    h += mix64(s[t] + (base + t) * kGold);
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)h);
}

// ---------------------------------------------------------------------------
// Exact centred basis conversion
// ---------------------------------------------------------------------------
// Rare path: decide v vs v+1 exactly by comparing 2X with (2v+1)B in
// multiword arithmetic (B odd => never equal).  X = sum xt_i * (B/b_i).
__device__ __noinline__ u64 tie_resolve(const ConvPlanDev* __restrict__ pl, const u64* __restrict__ hat_big,
                                        const u64* xt, u32 k, u64 v) {
  const u32 W = pl->big_words;
  u64 X[kMaxBigWords + 2];
  u64 R[kMaxBigWords + 2];
  for (u32 w = 0; w < W + 2; ++w) X[w] = R[w] = 0;
  for (u32 i = 0; i < k; ++i) {
    u64 carry = 0;
    for (u32 w = 0; w < W; ++w) {
      const u64 h = hat_big[(size_t)i * W + w];
      const u64 lo = h * xt[i], hi = __umul64hi(h, xt[i]);
      u64 s = X[w] + lo;
      u64 c1 = s < lo;
      s += carry;
      c1 += s < carry;
      X[w] = s;
      carry = hi + c1;
    }
    for (u32 w = W; w < W + 2 && carry; ++w) {
      X[w] += carry;
      carry = X[w] < carry;
    }
  }
  // X *= 2
  u64 top = 0;
  for (u32 w = 0; w < W + 2; ++w) {
    const u64 nt = X[w] >> 63;
    X[w] = (X[w] << 1) | top;
    top = nt;
  }
  // R = (2v+1) * B
  const u64 mlt = 2 * v + 1;
  u64 carry = 0;
  for (u32 w = 0; w < W; ++w) {
    const u64 lo = pl->b_big[w] * mlt, hi = __umul64hi(pl->b_big[w], mlt);
    u64 s = lo + carry;
    carry = hi + (s < lo);
    R[w] = s;
  }
  R[W] = carry;
  for (int w = (int)W + 1; w >= 0; --w) {
    if (X[w] != R[w]) return X[w] > R[w] ? v + 1 : v;
  }
  return v;  // unreachable (B odd)
}

template <int K>
__global__ void __launch_bounds__(256) basis_convert_kernel(const ConvPlanDev* __restrict__ pl,
                                                            const u64* __restrict__ hat_tab, const ConvIO io,
                                                            u32 lanes, u32 n, u32 kdyn, u32 m) {
  const u32 k = K > 0 ? (u32)K : kdyn;
  const u32 gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= lanes * n) return;
  const u32 lane = gid / n, x = gid - lane * n;
  const u64* src = io.src + (size_t)lane * io.src_lane_stride + x;
  u64* dst = io.dst + (size_t)lane * io.dst_lane_stride + x;
  constexpr int KA = K > 0 ? K : kMaxConv;
  u64 xt[KA];
  u64 F_lo = 0, F_hi = 0;
#pragma unroll
  for (u32 i = 0; i < (u32)KA; ++i) {
    if (i >= k) break;
    const u64 b = pl->src_p[i];
    const u64 t = shoup(src[(size_t)io.src_off[i] * n], pl->hat_inv[i], pl->hat_inv_p[i], b);
    xt[i] = t;
    const u64 f = t * pl->w_hi[i] + __umul64hi(t, pl->w_lo[i]);
    F_lo += f;
    F_hi += F_lo < f;
  }
  // v = round(F / 2^64); ambiguous when the fraction is within 2k ulps below 1/2
  const u64 half = 1ull << 63;
  u64 low = F_lo + half;
  u64 v = F_hi + (low < half);
  if (low >= (u64)0 - 2ull * k) v = tie_resolve(pl, hat_tab + (size_t)2 * k * m, xt, k, v);
  const u64* hm = hat_tab;  // [k][m]: (B/b_i) mod d_t
  Split xs[KA];
#pragma unroll
  for (u32 i = 0; i < (u32)KA; ++i) {
    if (i >= k) break;
    xs[i] = split24(xt[i]);
  }
  const Split vs = split24(v);
  for (u32 t = 0; t < m; ++t) {
    const u64 d = pl->dst_p[t];
    // sum_i xt_i [B/b_i]_d + v (d - [B]_d)  ==  x_centred mod d
    Acc3 s;
#pragma unroll
    for (u32 i = 0; i < (u32)KA; ++i) {
      if (i >= k) break;
      mac24(s, xs[i], split24(__ldg(hm + i * m + t)));
    }
    mac24(s, vs, split24(d - pl->b_mod[t]));
    dst[(size_t)io.dst_off[t] * n] = acc3_reduce(s, d, pl->dst_mu[t]);
  }
}

// First half of the conversion, once per source set: the
// sources are replaced in place by xt_i = x_i (B/b_i)^{-1} mod b_i and the
// overflow count v = round(sum xt_i / b_i) is written to vbuf.  The fused
// conversion + NTT pass (ntt.cu cfwd_a) then needs only k+1 MACs per target.
// one source coefficient x of `lane`: x~_i in place (split form) and v
template <int K>
__device__ __forceinline__ void conv_prep_one(const ConvPlanDev* __restrict__ pl, const u64* __restrict__ hat_tab,
                                              u32 m, const u64 (&raw)[K], u64 (&xt)[K], u64& v) {
  u64 F_lo = 0, F_hi = 0;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const u64 b = pl->src_p[i];
    const u64 t = shoup(raw[i], pl->hat_inv[i], pl->hat_inv_p[i], b);
    xt[i] = t;
    const u64 f = t * pl->w_hi[i] + __umul64hi(t, pl->w_lo[i]);
    F_lo += f;
    F_hi += F_lo < f;
  }
  const u64 half = 1ull << 63;
  u64 low = F_lo + half;
  v = F_hi + (low < half);
  if (low >= (u64)0 - 2ull * K) v = tie_resolve(pl, hat_tab + (size_t)2 * K * m, xt, K, v);
}

// two consecutive coefficients per thread (128-bit loads / stores: twice the
// bytes in flight of the one-coefficient form, which was latency-bound)
template <int K>
__global__ void __launch_bounds__(256) conv_prep_kernel(const ConvPlanDev* __restrict__ pl,
                                                        const u64* __restrict__ hat_tab, ConvIO io, u64* vbuf,
                                                        size_t v_ls, u32 lanes, u32 n, u32 m) {
  pdl_wait();
  const u32 gid = blockIdx.x * blockDim.x + threadIdx.x;
  const u32 half_n = n / 2;
  if (gid >= lanes * half_n) return;
  const u32 lane = gid / half_n, x = (gid - lane * half_n) * 2;
  u64* src = const_cast<u64*>(io.src) + (size_t)lane * io.src_lane_stride + x;
  u64 ra[K], rb[K];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(src + (size_t)io.src_off[i] * n);
    ra[i] = w.x;
    rb[i] = w.y;
  }
  u64 xa[K], xb[K], va, vb;
  conv_prep_one<K>(pl, hat_tab, m, ra, xa, va);
  conv_prep_one<K>(pl, hat_tab, m, rb, xb, vb);
#pragma unroll
  for (int i = 0; i < K; ++i)
    *reinterpret_cast<ulonglong2*>(src + (size_t)io.src_off[i] * n) =
        make_ulonglong2((xa[i] & 0xFFFFFFull) | ((xa[i] >> 24) << 32), (xb[i] & 0xFFFFFFull) | ((xb[i] >> 24) << 32));
  // v <= k < 2^24: already in split form
  *reinterpret_cast<ulonglong2*>(vbuf + (size_t)lane * v_ls + x) = make_ulonglong2(va, vb);
}

// ---------------------------------------------------------------------------
// Key inner product
// ---------------------------------------------------------------------------
__global__ void keymul_kernel(const KeyMulIO io, u32 lanes, u32 n, const PrimeConst* __restrict__ pc,
                              u32 cpr) {
  // lanes vary fastest across the grid: CTAs running together share the key
  // limbs of one slot, so a batch streams each key limb from HBM once (L2 hits
  // for the other lanes) instead of once per lane.
  const u32 lane = blockIdx.x % lanes, rest = blockIdx.x / lanes;
  const u32 chunk = rest % cpr, slot = rest / cpr;
  const u32 e = io.slot_ext[slot];
  const PrimeConst P = pc[e];
  const u32 ks = io.slot_key[slot];
  const size_t kslot_stride = (size_t)io.key_slots * n;  // per comp
  const u64* dd = io.d + (size_t)lane * io.d_lane_stride + (size_t)slot * n;
  u64* a0 = io.acc + (size_t)lane * io.acc_lane_stride + (size_t)slot * n;
  u64* a1 = a0 + (size_t)io.nslots * n;
  const bool main_slot = slot < io.level;
  for (u32 x = chunk * kChunk + threadIdx.x; x < n && x < (chunk + 1) * kChunk; x += kThreads) {
    Acc3 s0, s1;
    for (u32 j = 0; j < io.dnum; ++j) {
      const u32 lo = j * kAlpha, hi = lo + kAlpha < io.level ? lo + kAlpha : io.level;
      const bool own = main_slot && slot >= lo && slot < hi;
      // compact ModUp layout (Context::modup_words_per_lane): digit j at (j*ns - lo)
      const u32 idx = j * io.nslots - lo + (slot < lo ? slot : slot - (hi - lo));
      const Split v = split24(own ? dd[x] : io.ext[(size_t)lane * io.ext_lane_stride + (size_t)idx * n + x]);
      const u64* kj = io.key + (size_t)j * 2 * kslot_stride + (size_t)ks * n + x;
      mac24(s0, v, split24(__ldg(kj)));
      mac24(s1, v, split24(__ldg(kj + kslot_stride)));
    }
    a0[x] = acc3_reduce(s0, P.p, P.mu104);
    a1[x] = acc3_reduce(s1, P.p, P.mu104);
  }
}

// Key product with every load of a coefficient issued up front: DN ext/d
// words and 2*DN key words per thread are in flight together (the looped
// form exposes one memory latency per digit).  Lanes vary fastest across the
// grid so CTAs in flight share the key tile of one (slot, chunk) in L2.
// Two adjacent coefficients per thread (128-bit loads and stores) for the
// FP64 key product at DN <= 5 (the hoisted rotations at level 17): half the
// load instructions for the same bytes in flight.
template <int DN>
__global__ void __launch_bounds__(256) keymul_dn2_kernel(const KeyMulIO io, u32 lanes, u32 n,
                                                         const PrimeConst* __restrict__ pc) {
  pdl_wait();
  const u32 chunks = n / 512;
  const u32 lane = blockIdx.x % lanes, rest = blockIdx.x / lanes;
  const u32 chunk = rest % chunks, slot = rest / chunks;
  const u32 x = (chunk * 256 + threadIdx.x) * 2;
  const PrimeConst P = pc[io.slot_ext[slot]];
  const size_t kslot_stride = (size_t)io.key_slots * n;
  const u64* kb = io.key + (size_t)io.slot_key[slot] * n + x;
  const u64* eb = io.ext + (size_t)lane * io.ext_lane_stride + x;
  const u64* db = io.d + (size_t)lane * io.d_lane_stride + (size_t)slot * n + x;
  const bool main_slot = slot < io.level;
  ulonglong2 e[DN], k0[DN], k1[DN];
  u32 own_mask = 0;
#pragma unroll
  for (int j = 0; j < DN; ++j) {
    const u32 lo = j * kAlpha, hi = lo + kAlpha < io.level ? lo + kAlpha : io.level;
    const bool own = main_slot && slot >= lo && slot < hi;
    own_mask |= own ? 1u << j : 0u;
    const u32 idx = j * io.nslots - lo + (slot < lo ? slot : slot - (hi - lo));
    e[j] = *reinterpret_cast<const ulonglong2*>(own ? db : eb + (size_t)idx * n);
    k0[j] = __ldg(reinterpret_cast<const ulonglong2*>(kb + (size_t)j * 2 * kslot_stride));
    k1[j] = __ldg(reinterpret_cast<const ulonglong2*>(kb + (size_t)j * 2 * kslot_stride + kslot_stride));
  }
  const double pd = f64_of(P.p), pinv = 1.0 / pd;
  double s0a = 0.0, s0b = 0.0, s1a = 0.0, s1b = 0.0;
#pragma unroll
  for (int j = 0; j < DN; ++j) {
    const bool lazy = io.ext_lazy && !(own_mask >> j & 1u);
    const double va = lazy ? __longlong_as_double((long long)e[j].x) : f64_of(e[j].x);
    const double vb = lazy ? __longlong_as_double((long long)e[j].y) : f64_of(e[j].y);
    const double w0a = f64_of(k0[j].x), w0b = f64_of(k0[j].y), w1a = f64_of(k1[j].x), w1b = f64_of(k1[j].y);
    s0a += f64_mulmod(va, w0a, w0a * pinv, pd);
    s0b += f64_mulmod(vb, w0b, w0b * pinv, pd);
    s1a += f64_mulmod(va, w1a, w1a * pinv, pd);
    s1b += f64_mulmod(vb, w1b, w1b * pinv, pd);
  }
  u64* a0 = io.acc + (size_t)lane * io.acc_lane_stride + (size_t)slot * n + x;
  *reinterpret_cast<ulonglong2*>(a0) = make_ulonglong2(f64_canon(s0a, pd, pinv), f64_canon(s0b, pd, pinv));
  *reinterpret_cast<ulonglong2*>(a0 + (size_t)io.nslots * n) =
      make_ulonglong2(f64_canon(s1a, pd, pinv), f64_canon(s1b, pd, pinv));
}

template <int DN, bool F64>
__global__ void __launch_bounds__(256) keymul_dn_kernel(const KeyMulIO io, u32 lanes, u32 n,
                                                        const PrimeConst* __restrict__ pc) {
  const u32 chunks = n / 256;
  const u32 lane = blockIdx.x % lanes, rest = blockIdx.x / lanes;
  const u32 chunk = rest % chunks, slot = rest / chunks;
  const u32 x = chunk * 256 + threadIdx.x;
  const PrimeConst P = pc[io.slot_ext[slot]];
  const size_t kslot_stride = (size_t)io.key_slots * n;
  const u64* kb = io.key + (size_t)io.slot_key[slot] * n + x;
  const u64* eb = io.ext + (size_t)lane * io.ext_lane_stride + x;
  const u64* db = io.d + (size_t)lane * io.d_lane_stride + (size_t)slot * n + x;
  const bool main_slot = slot < io.level;
  u64 e[DN], k0[DN], k1[DN];
  u32 own_mask = 0;
#pragma unroll
  for (int j = 0; j < DN; ++j) {
    const u32 lo = j * kAlpha, hi = lo + kAlpha < io.level ? lo + kAlpha : io.level;
    const bool own = main_slot && slot >= lo && slot < hi;
    own_mask |= own ? 1u << j : 0u;
    const u32 idx = j * io.nslots - lo + (slot < lo ? slot : slot - (hi - lo));
    e[j] = own ? db[0] : eb[(size_t)idx * n];
    k0[j] = __ldg(kb + (size_t)j * 2 * kslot_stride);
    k1[j] = __ldg(kb + (size_t)j * 2 * kslot_stride + kslot_stride);
  }
  u64* a0 = io.acc + (size_t)lane * io.acc_lane_stride + (size_t)slot * n + x;
  if constexpr (!F64) {
    Acc3 s0, s1;
#pragma unroll
    for (int j = 0; j < DN; ++j) {
      const Split v = split24(e[j]);
      mac24(s0, v, split24(k0[j]));
      mac24(s1, v, split24(k1[j]));
    }
    a0[0] = acc3_reduce(s0, P.p, P.mu104);
    a0[(size_t)io.nslots * n] = acc3_reduce(s1, P.p, P.mu104);
    return;
  }
  // exact FP64 products on the otherwise idle DFMA pipe (the 24-bit integer
  // MACs make this kernel ALU-bound); DN terms in [-1.5p, 1.5p] sum exactly
  const double pd = f64_of(P.p), pinv = 1.0 / pd;
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int j = 0; j < DN; ++j) {
    // own-digit words are canonical u64 (d); ModUp words may be lazy FP64 bits
    const bool lazy = io.ext_lazy && !(own_mask >> j & 1u);
    const double v = lazy ? __longlong_as_double((long long)e[j]) : f64_of(e[j]);
    const double w0 = f64_of(k0[j]), w1 = f64_of(k1[j]);
    s0 += f64_mulmod(v, w0, w0 * pinv, pd);
    s1 += f64_mulmod(v, w1, w1 * pinv, pd);
  }
  a0[0] = f64_canon(s0, pd, pinv);
  a0[(size_t)io.nslots * n] = f64_canon(s1, pd, pinv);
}

__global__ void finish_kernel(const FinishIO io, u32 n, const PrimeConst* __restrict__ pc, u32 cpr) {
  const u32 row = blockIdx.x / cpr, chunk = blockIdx.x - row * cpr;
  const u32 lb = row % io.limbs, rest = row / io.limbs, comp = rest % io.comps, lane = rest / io.comps;
  const u64 p = pc[io.ext[lb]].p;
  const u64 f = io.f[lb], fp = io.f_p[lb];
  const u64* x = io.x + lane * io.x_lane + comp * io.x_comp + (size_t)lb * n;
  const u64* y = io.y + lane * io.y_lane + comp * io.y_comp + (size_t)lb * n;
  const u64* ad = io.add ? io.add + lane * io.add_lane + comp * io.add_comp + (size_t)lb * n : nullptr;
  u64* o = io.out + lane * io.out_lane + comp * io.out_comp + (size_t)lb * n;
  const u32 mask = 2 * n - 1, k = (u32)(io.galois & mask);
  const int sh = 32 - (int)io.log_n;
  for (u32 t = chunk * kChunk + threadIdx.x; t < n && t < (chunk + 1) * kChunk; t += kThreads) {
    // optional eval-domain automorphism of the result: read position pi(t)
    // (maps aligned 32-blocks onto aligned 32-blocks, so the gather coalesces)
    u32 s = t;
    if (k > 1) s = __brev(((((__brev(t) >> sh) * 2 + 1) * k & mask) - 1) >> 1) >> sh;
    u64 r = shoup(sub_mod(x[s], y[s], p), f, fp, p);
    if (ad) r = add_mod(r, ad[s], p);
    o[t] = r;
  }
}

// ---------------------------------------------------------------------------
// Bundled PCMM step with in-kernel weights (kGenerate, poly_ir.hpp:57, 310-321)
// ---------------------------------------------------------------------------
constexpr u32 kPmTx = 32;      // coefficients per CTA
constexpr u32 kPmGroups = 8;   // max o-groups per CTA (256 threads)

// o-groups per CTA: the largest divisor of c_out <= kPmGroups, so every
// thread runs the same number of outputs (c_out = 12 -> 6 groups x 2)
inline u32 pmult_groups(u32 c_out) {
  for (u32 g = kPmGroups; g > 1; --g)
    if (c_out % g == 0) return g;
  return c_out < kPmGroups ? c_out : kPmGroups;
}

// acc lane for (token group t, output o') is acc_lane0 + t*c_out + o'; the
// weight lane is ci*w_cout + o_off + o' (o_off/w_cout select one sub-tensor
// of a chunked accumulator, CtBundle::chunk_period, he_ir.hpp:338).
// SMEM: x tile pre-split into 24-bit limbs [TG * c_in][2][kPmTx], then this
// limb's weight row keys [c_in][c_out] (read once per (ci, o) by a warp, so
// the per-iteration key fetch is an LDS broadcast, not a dependent LDG).
// MINB: resident CTAs the register budget targets -- 3 when SMEM allows it
// (TG = 4 then spills a few words, still the faster trade), else 2.
template <int TG, int MINB, bool STORED>
__global__ void __launch_bounds__(256, MINB) pmult_kernel(const PmultArgs a, const PrimeConst* __restrict__ pc) {
  extern __shared__ Split xs[];
  const u32 n = a.n, c_in = a.c_in, c_out = a.c_out, limbs = a.limbs;
  const u32 tiles = n / kPmTx;
  const u32 lb = blockIdx.x / tiles;
  const u32 x0 = (blockIdx.x - lb * tiles) * kPmTx;
  const PrimeConst P = pc[lb];
  const u32 nx = TG * c_in;
  u64* rks = reinterpret_cast<u64*>(xs + nx * 2 * kPmTx);
  if (!STORED)
    for (u32 e = threadIdx.x; e < c_in * c_out; e += blockDim.x) {
      const u32 ci = e / c_out, o = e - ci * c_out;
      rks[e] = a.rowkeys[(size_t)((a.ci_off + ci) * a.w_cout + a.o_off + o) * limbs + lb];
    }
  for (u32 e = threadIdx.x; e < nx * 2 * kPmTx; e += blockDim.x) {
    const u32 xx = e % kPmTx, r = e / kPmTx, comp = r & 1, ln = r >> 1;
    const u32 t = ln / c_in, ci = ln - t * c_in;
    xs[e] = split24(a.x.limb(a.x_lane0 + t * a.x_tstride + ci, comp, lb, n)[x0 + xx]);
  }
  __syncthreads();
  const u32 groups = blockDim.x / kPmTx;
  const u32 xx = threadIdx.x % kPmTx;
  const u32 og = threadIdx.x / kPmTx;
  const u64 xi = x0 + xx;
  for (u32 o = og; o < c_out; o += groups) {
    // the accumulator words are fetched before the MAC loop so their latency
    // hides under it (the loads cannot move across the stores otherwise)
    u64 prev[TG][2];
#pragma unroll
    for (int t = 0; t < TG; ++t)
#pragma unroll
      for (int cp = 0; cp < 2; ++cp) prev[t][cp] = a.acc.limb(a.acc_lane0 + t * a.acc_tstride + o, cp, lb, n)[xi];
    Acc3 s[TG][2];
#pragma unroll 1
    for (u32 ci = 0; ci < c_in; ++ci) {
      const Split w = STORED ? split24(a.wst.limb(a.w_lane0 + (a.ci_off + ci) * a.w_cout + a.o_off + o, 0, lb, n)[xi])
                             : split24(uniform_at(rks[ci * c_out + o], xi, P.p, P.shift));
#pragma unroll
      for (int t = 0; t < TG; ++t) {
        const u32 r = (t * c_in + ci) * 2;
        mac24_ptx(s[t][0], xs[r * kPmTx + xx], w);
        mac24_ptx(s[t][1], xs[(r + 1) * kPmTx + xx], w);
      }
    }
#pragma unroll
    for (int t = 0; t < TG; ++t)
#pragma unroll
      for (int cp = 0; cp < 2; ++cp) {
        s[t][cp].c0 += prev[t][cp];
        a.acc.limb(a.acc_lane0 + t * a.acc_tstride + o, cp, lb, n)[xi] = acc3_reduce(s[t][cp], P.p, P.mu104);
      }
  }
}

__global__ void weight_rowkeys_kernel(u64* out, u32 wlanes, u32 limbs, u64 seed, u64 bundle) {
  const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= wlanes * limbs) return;
  const u32 lane = i / limbs, lb = i - lane * limbs;
  out[i] = row_key(seed, 2, bundle, lane, 0, lb);  // tag 2: generated weights
}

}  // namespace

int g_km_f64 = 1;

// ---------------------------------------------------------------------------
// launch wrappers
// ---------------------------------------------------------------------------
cudaError_t launch_fill_uniform(View v, u32 lanes, u32 comps, u32 limbs, u32 n, u64 seed, u64 tag,
                                u64 a, const u32* limb_ext, const PrimeConst* pc, cudaStream_t st) {
  const u32 cpr = chunks_of(n);
  const size_t g = (size_t)lanes * comps * limbs * cpr;
  if (!g) return cudaSuccess;
  fill_uniform_kernel<<<(unsigned)g, kThreads, 0, st>>>(v, comps, limbs, n, seed, tag, a, limb_ext, pc, cpr);
  return cudaGetLastError();
}

cudaError_t launch_fill_key(u64* key, u32 digits, u32 slots, u32 n, u64 seed, u64 key_id,
                            const u32* slot_ext, const PrimeConst* pc, cudaStream_t st) {
  const u32 cpr = chunks_of(n);
  const size_t g = (size_t)digits * 2 * slots * cpr;
  fill_key_kernel<<<(unsigned)g, kThreads, 0, st>>>(key, slots, n, seed, key_id, slot_ext, pc, cpr);
  return cudaGetLastError();
}

cudaError_t launch_automorphism(View out, LaneMap om, View in, LaneMap im, u32 nlanes, u32 comps,
                                u32 limbs, u32 log_n, u64 galois, cudaStream_t st) {
  const u32 n = 1u << log_n;
  const u32 cpr = chunks_of(n);
  const size_t g = (size_t)nlanes * comps * limbs * cpr;
  if (!g) return cudaSuccess;
  automorphism_kernel<<<(unsigned)g, kThreads, 0, st>>>(out, om, in, im, nlanes, comps, limbs, log_n,
                                                         galois, cpr);
  return cudaGetLastError();
}

cudaError_t launch_cmult(View out, u32 out_lane0, View a, LaneMap ma, View b, LaneMap mb, u32 nlanes,
                         u32 limbs, u32 n, const PrimeConst* pc, cudaStream_t st) {
  if (n % 1024 == 0) {
    const size_t g = (size_t)nlanes * limbs * (n / 1024);
    if (!g) return cudaSuccess;
    const bool square = a.base == b.base && a.comps == b.comps && a.levels == b.levels && ma.lane0 == mb.lane0 &&
                        ma.count == mb.count;
    if (square)
      square4_kernel<<<(unsigned)g, 256, 0, st>>>(out, out_lane0, a, ma, nlanes, limbs, n, pc);
    else
      cmult4_kernel<<<(unsigned)g, 256, 0, st>>>(out, out_lane0, a, ma, b, mb, nlanes, limbs, n, pc);
    return cudaGetLastError();
  }
  const u32 cpr = chunks_of(n);
  const size_t g = (size_t)nlanes * limbs * cpr;
  if (!g) return cudaSuccess;
  cmult_kernel<<<(unsigned)g, kThreads, 0, st>>>(out, out_lane0, a, ma, b, mb, nlanes, limbs, n, pc, cpr);
  return cudaGetLastError();
}

cudaError_t launch_cadd(View out, u32 out_lane0, View a, LaneMap ma, View b, LaneMap mb, bool acc,
                        u32 nlanes, u32 comps, u32 limbs, u32 n, const PrimeConst* pc, cudaStream_t st) {
  const u32 cpr = (n + 2047) / 2048;
  const size_t g = (size_t)nlanes * comps * limbs * cpr;
  if (!g) return cudaSuccess;
  cadd_kernel<<<(unsigned)g, kThreads, 0, st>>>(out, out_lane0, a, ma, b, mb, acc ? 1 : 0, nlanes, comps,
                                                 limbs, n, pc, cpr);
  return cudaGetLastError();
}

cudaError_t launch_copy(View dst, u32 dst_lane0, View src, LaneMap sm, u32 nlanes, u32 comps, u32 limbs,
                        u32 src_limb0, u32 n, cudaStream_t st) {
  const u32 cpr = chunks_of(n);
  const size_t g = (size_t)nlanes * comps * limbs * cpr;
  if (!g) return cudaSuccess;
  copy_kernel<<<(unsigned)g, kThreads, 0, st>>>(dst, dst_lane0, src, sm, nlanes, comps, limbs, src_limb0, n,
                                                 cpr);
  return cudaGetLastError();
}

cudaError_t launch_hash(View v, u32 lane0, u32 lanes, u32 comps, u32 limbs, u32 n, unsigned long long* out,
                        cudaStream_t st) {
  const u32 cpr = chunks_of(n);
  const size_t g = (size_t)lanes * comps * limbs * cpr;
  if (!g) return cudaSuccess;
  hash_kernel<<<(unsigned)g, kThreads, 0, st>>>(v, lane0, comps, limbs, n, out, cpr);
  return cudaGetLastError();
}

// values < 2^64 of lanes [lane0, lane0+lanes), comps x limbs -> canonical (after a uint64 reduce-scatter)
__global__ void reduce_lanes_kernel(View v, u32 lane0, u32 comps, u32 limbs, u32 n,
                                    const PrimeConst* __restrict__ pc, u32 cpr) {
  const u32 row = blockIdx.x / cpr, chunk = blockIdx.x - row * cpr;
  const u32 lb = row % limbs, rest = row / limbs, comp = rest % comps, lane = lane0 + rest / comps;
  const PrimeConst P = pc[lb];
  u64* s = v.limb(lane, comp, lb, n);
  for (u32 t = chunk * kChunk + threadIdx.x; t < n && t < (chunk + 1) * kChunk; t += kThreads)
    s[t] = reduce104(u128{s[t], 0}, P.p, P.mu104);
}

cudaError_t launch_reduce_lanes(View v, u32 lane0, u32 lanes, u32 comps, u32 limbs, u32 n, const PrimeConst* pc,
                                cudaStream_t st) {
  const u32 cpr = chunks_of(n);
  const size_t g = (size_t)lanes * comps * limbs * cpr;
  if (!g) return cudaSuccess;
  reduce_lanes_kernel<<<(unsigned)g, kThreads, 0, st>>>(v, lane0, comps, limbs, n, pc, cpr);
  return cudaGetLastError();
}

cudaError_t launch_basis_convert(const ConvPlanDev* plan, const u64* hat_tables, const ConvIO& io,
                                 u32 lanes, u32 n, u32 k, u32 m, cudaStream_t st) {
  const size_t total = (size_t)lanes * n;
  if (!total) return cudaSuccess;
  const unsigned grid = (unsigned)((total + 255) / 256);
  switch (k) {
    case 1: basis_convert_kernel<1><<<grid, 256, 0, st>>>(plan, hat_tables, io, lanes, n, k, m); break;
    case 2: basis_convert_kernel<2><<<grid, 256, 0, st>>>(plan, hat_tables, io, lanes, n, k, m); break;
    case 3: basis_convert_kernel<3><<<grid, 256, 0, st>>>(plan, hat_tables, io, lanes, n, k, m); break;
    case 4: basis_convert_kernel<4><<<grid, 256, 0, st>>>(plan, hat_tables, io, lanes, n, k, m); break;
    default: basis_convert_kernel<0><<<grid, 256, 0, st>>>(plan, hat_tables, io, lanes, n, k, m); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_conv_prep(const ConvPlanDev* plan, const u64* hat_tables, const ConvIO& io, u64* vbuf,
                             size_t v_ls, u32 lanes, u32 n, u32 k, u32 m, cudaStream_t st) {
  const size_t total = (size_t)lanes * (n / 2);
  if (!total) return cudaSuccess;
  const unsigned grid = (unsigned)((total + 255) / 256);
  switch (k) {
    case 1: launch_pdl(conv_prep_kernel<1>, dim3(grid), dim3(256), 0, st, plan, hat_tables, io, vbuf, v_ls, lanes, n, m); break;
    case 2: launch_pdl(conv_prep_kernel<2>, dim3(grid), dim3(256), 0, st, plan, hat_tables, io, vbuf, v_ls, lanes, n, m); break;
    case 3: launch_pdl(conv_prep_kernel<3>, dim3(grid), dim3(256), 0, st, plan, hat_tables, io, vbuf, v_ls, lanes, n, m); break;
    case 4: launch_pdl(conv_prep_kernel<4>, dim3(grid), dim3(256), 0, st, plan, hat_tables, io, vbuf, v_ls, lanes, n, m); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_keymul(const KeyMulIO& io, u32 lanes, u32 n, const PrimeConst* pc, cudaStream_t st) {
  if (g_km_f64 && n >= 512 && io.dnum >= 1 && io.dnum <= 9) {
    const size_t g = (size_t)lanes * io.nslots * (n / 512);
    switch (io.dnum) {
      case 1: launch_pdl(keymul_dn2_kernel<1>, dim3((unsigned)g), dim3(256), 0, st, io, lanes, n, pc); break;
      case 2: launch_pdl(keymul_dn2_kernel<2>, dim3((unsigned)g), dim3(256), 0, st, io, lanes, n, pc); break;
      case 3: launch_pdl(keymul_dn2_kernel<3>, dim3((unsigned)g), dim3(256), 0, st, io, lanes, n, pc); break;
      case 4: launch_pdl(keymul_dn2_kernel<4>, dim3((unsigned)g), dim3(256), 0, st, io, lanes, n, pc); break;
      case 5: launch_pdl(keymul_dn2_kernel<5>, dim3((unsigned)g), dim3(256), 0, st, io, lanes, n, pc); break;
      case 6: launch_pdl(keymul_dn2_kernel<6>, dim3((unsigned)g), dim3(256), 0, st, io, lanes, n, pc); break;
      case 7: launch_pdl(keymul_dn2_kernel<7>, dim3((unsigned)g), dim3(256), 0, st, io, lanes, n, pc); break;
      case 8: launch_pdl(keymul_dn2_kernel<8>, dim3((unsigned)g), dim3(256), 0, st, io, lanes, n, pc); break;
      default: launch_pdl(keymul_dn2_kernel<9>, dim3((unsigned)g), dim3(256), 0, st, io, lanes, n, pc); break;
    }
    return cudaGetLastError();
  }
  if (n >= 256 && io.dnum >= 1 && io.dnum <= 9) {
    const size_t g = (size_t)lanes * io.nslots * (n / 256);
#define AEGIS_KM(D) \
  case D:                                                                                       \
    if (g_km_f64) keymul_dn_kernel<D, true><<<(unsigned)g, 256, 0, st>>>(io, lanes, n, pc);      \
    else keymul_dn_kernel<D, false><<<(unsigned)g, 256, 0, st>>>(io, lanes, n, pc);              \
    break;
    switch (io.dnum) {
      AEGIS_KM(1) AEGIS_KM(2) AEGIS_KM(3) AEGIS_KM(4) AEGIS_KM(5) AEGIS_KM(6) AEGIS_KM(7) AEGIS_KM(8) AEGIS_KM(9)
    }
#undef AEGIS_KM
    return cudaGetLastError();
  }
  const u32 cpr = chunks_of(n);
  const size_t g = (size_t)lanes * io.nslots * cpr;
  if (!g) return cudaSuccess;
  keymul_kernel<<<(unsigned)g, kThreads, 0, st>>>(io, lanes, n, pc, cpr);
  return cudaGetLastError();
}

cudaError_t launch_finish(const FinishIO& io, u32 lanes, u32 n, const PrimeConst* pc, cudaStream_t st) {
  const u32 cpr = chunks_of(n);
  const size_t g = (size_t)lanes * io.comps * io.limbs * cpr;
  if (!g) return cudaSuccess;
  finish_kernel<<<(unsigned)g, kThreads, 0, st>>>(io, n, pc, cpr);
  return cudaGetLastError();
}

cudaError_t launch_weight_rowkeys(u64* out, u32 wlanes, u32 limbs, u64 seed, u64 bundle, cudaStream_t st) {
  const u32 total = wlanes * limbs;
  if (!total) return cudaSuccess;
  weight_rowkeys_kernel<<<(total + 255) / 256, 256, 0, st>>>(out, wlanes, limbs, seed, bundle);
  return cudaGetLastError();
}

cudaError_t launch_pmult_acc(const PmultArgs& a, const PrimeConst* pc, cudaStream_t st) {
  if (a.n < kPmTx) return cudaErrorInvalidValue;
  const u32 tg4 = a.tg < 4 ? a.tg : 4;
  const bool stored = a.wst.base != nullptr;
  const size_t smem = ((size_t)tg4 * a.c_in * 2 * kPmTx + (stored ? 0 : (size_t)a.c_in * a.c_out)) * sizeof(u64);
  const unsigned grid = a.limbs * (a.n / kPmTx);
  const unsigned block = kPmTx * pmult_groups(a.c_out);
  if (!grid || !a.c_in || !a.c_out) return cudaSuccess;
#define AEGIS_PM(TGV)                                                                          \
  case TGV: {                                                                                  \
    auto kern = stored ? (smem * 3 <= 220 * 1024 ? pmult_kernel<TGV, 3, true> : pmult_kernel<TGV, 2, true>)    \
                       : (smem * 3 <= 220 * 1024 ? pmult_kernel<TGV, 3, false> : pmult_kernel<TGV, 2, false>); \
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    kern<<<grid, block, smem, st>>>(a, pc);                                        \
    break;                                                                                     \
  }
  switch (a.tg) {
    AEGIS_PM(1)
    AEGIS_PM(2)
    AEGIS_PM(3)
    AEGIS_PM(4)
    default: {
      // more token groups than the templated cases: process in groups of 4
      for (u32 t0 = 0; t0 < a.tg; t0 += 4) {
        PmultArgs b = a;
        b.tg = a.tg - t0 < 4 ? a.tg - t0 : 4;
        b.acc_lane0 = a.acc_lane0 + t0 * a.acc_tstride;
        b.x_lane0 = a.x_lane0 + t0 * a.x_tstride;
        cudaError_t e = launch_pmult_acc(b, pc, st);
        if (e != cudaSuccess) return e;
      }
      return cudaSuccess;
    }
  }
#undef AEGIS_PM
  return cudaGetLastError();
}

}  // namespace aegis

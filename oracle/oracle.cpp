// oracle/oracle.cpp -- TEST INFRASTRUCTURE ONLY: the CPU checker for libaegis.
//
// A plain, scalar C++ restatement of the reference's arithmetic and of the
// HE-op semantics pinned in DESIGN.md §2.  Nothing here is shared with the
// product library except the prime table (include/aegis_params.h, data only).
// Reference anchors (relative to /root/reference/proj/include/heplan/):
//   mod ops            rns_math.hpp:21-40
//   NTT tables / psi   rns_math.hpp:46-63, 103-117
//   forward / inverse  rns_math.hpp:68-100
//   automorphism       rns_math.hpp:127-149
//   centred CRT        rns_math.hpp:151-193  (restated exactly at any size)
//   div_round          rns_math.hpp:196-202  (rescale / ModDown rounding)
//   key switch         poly_ir.hpp:219-305   (Intt/Auto/ModUp/KeyMul/ModDown/Ntt)
//   HE-op lane rules   he_ir.hpp:200-222 (emit_per_lane), 426-452, 328-373
//   exec_sequential
#include "oracle.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include <omp.h>
#include <sys/mman.h>

#include "../include/aegis_params.h"

typedef unsigned __int128 u128;
typedef uint64_t u64;
typedef uint32_t u32;

static thread_local std::string g_err;

namespace {

constexpr u64 kGold = 0x9E3779B97F4A7C15ULL;
constexpr u64 kMixM = 0xD6E8FEB86659FD93ULL;
constexpr u32 kSpecialBase = AEGIS_MAX_MAIN_PRIMES;  // ext index of P_0

u64 mix64(u64 x) {
  x ^= x >> 32;
  x *= kMixM;
  x ^= x >> 32;
  x *= kMixM;
  x ^= x >> 32;
  return x;
}

u64 row_key(u64 seed, u64 tag, u64 a, u64 b, u64 c, u64 d) {
  u64 k = mix64(seed ^ (tag * kGold));
  k = mix64(k ^ ((a + 1) * kGold));
  k = mix64(k ^ ((b + 1) * kGold));
  k = mix64(k ^ ((c + 1) * kGold));
  k = mix64(k ^ ((d + 1) * kGold));
  return k;
}

int bitlen(u64 p) { return 64 - __builtin_clzll(p); }

// uniform residue for coefficient i of a row
inline u64 uniform_at(u64 rk, u64 i, u64 p, int shift) {
  u64 v = mix64(rk + i * kGold) >> shift;
  return v >= p ? v - p : v;
}

inline u64 add_mod(u64 a, u64 b, u64 p) { u64 s = a + b; return s >= p ? s - p : s; }
inline u64 sub_mod(u64 a, u64 b, u64 p) { return a >= b ? a - b : a + p - b; }
inline u64 mul_mod(u64 a, u64 b, u64 p) { return (u64)(((u128)a * b) % p); }
u64 pow_mod(u64 b, u64 e, u64 p) {
  u64 r = 1 % p;
  b %= p;
  while (e) {
    if (e & 1) r = mul_mod(r, b, p);
    b = mul_mod(b, b, p);
    e >>= 1;
  }
  return r;
}
u64 inv_mod(u64 a, u64 p) { return pow_mod(a % p, p - 2, p); }
inline u64 shoup_pre(u64 w, u64 p) { return (u64)(((u128)w << 64) / p); }
inline u64 shoup_mul(u64 a, u64 w, u64 wp, u64 p) {
  u64 q = (u64)(((u128)a * wp) >> 64);
  u64 r = a * w - q * p;
  return r >= p ? r - p : r;
}

u32 bit_reverse(u32 v, int bits) {
  u32 r = 0;
  for (int i = 0; i < bits; ++i, v >>= 1) r = (r << 1) | (v & 1);
  return r;
}

// ---- multi-precision helpers (little-endian u64 words) -------------------
typedef std::vector<u64> Big;
void big_mul_small(Big& a, u64 m) {
  u64 carry = 0;
  for (auto& w : a) {
    u128 t = (u128)w * m + carry;
    w = (u64)t;
    carry = (u64)(t >> 64);
  }
  if (carry) a.push_back(carry);
}
void big_add(Big& a, const Big& b) {
  if (a.size() < b.size()) a.resize(b.size(), 0);
  u64 carry = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    u128 t = (u128)a[i] + (i < b.size() ? b[i] : 0) + carry;
    a[i] = (u64)t;
    carry = (u64)(t >> 64);
  }
  if (carry) a.push_back(carry);
}
void big_trim(Big& a) { while (a.size() > 1 && a.back() == 0) a.pop_back(); }
int big_cmp(Big a, Big b) {
  big_trim(a); big_trim(b);
  if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
  for (size_t i = a.size(); i-- > 0;)
    if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  return 0;
}
void big_sub(Big& a, const Big& b) {  // a >= b
  u64 borrow = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    u64 bi = i < b.size() ? b[i] : 0;
    u128 t = (u128)a[i] - bi - borrow;
    a[i] = (u64)t;
    borrow = (t >> 64) ? 1 : 0;
  }
  big_trim(a);
}
u64 big_mod_small(const Big& a, u64 p) {
  u128 r = 0;
  for (size_t i = a.size(); i-- > 0;) r = ((r << 64) | a[i]) % p;
  return (u64)r;
}

// ---- NTT tables (rns_math.hpp:46-63, 103-117) ----------------------------
struct NttTable {
  u64 p = 0, psi = 0, n_inv = 0, n_inv_p = 0;
  std::vector<u64> fwd, fwd_p, inv, inv_p;
};

// Exact centred basis conversion plan (rns_math.hpp:151-193, restated for any size).
struct ConvPlan {
  std::vector<u64> src_p, dst_p;
  std::vector<u64> hat_inv, hat_inv_p;     // (B/b_i)^{-1} mod b_i
  std::vector<u64> w_hi, w_lo;             // floor(2^128 / b_i)
  std::vector<u64> hat_mod;                // [i][t] (B/b_i) mod d_t
  std::vector<u64> b_mod;                  // [t] B mod d_t
  std::vector<Big> hat_big;                // B/b_i
  Big b_big;                               // B
};

}  // namespace

struct orc_ctx {
  u32 log_n, n, chain, lboot;
  u64 seed_input, seed_weight, seed_key;
  int threads;
  std::vector<u64> prime;  // by ext index (0..63)
  std::vector<int> shift;
  std::vector<std::unique_ptr<NttTable>> tables;
  std::mutex mu;
  std::map<std::vector<u32>, std::shared_ptr<ConvPlan>> plans;
  std::map<std::vector<u64>, std::shared_ptr<std::vector<u64>>> key_cache;

  const NttTable& table(u32 e) {
    std::lock_guard<std::mutex> g(mu);
    if (!tables[e]) tables[e] = build_table(prime[e]);
    return *tables[e];
  }
  std::unique_ptr<NttTable> build_table(u64 p) {
    auto t = std::make_unique<NttTable>();
    t->p = p;
    if ((p - 1) % (2ull * n) != 0) throw std::invalid_argument("prime does not support NTT");
    // psi: first g >= 2 whose g^((p-1)/2n) has order 2n (rns_math.hpp:103-111)
    const u64 order = 2ull * n;
    for (u64 g = 2; g < p; ++g) {
      u64 cand = pow_mod(g, (p - 1) / order, p);
      if (pow_mod(cand, n, p) == p - 1) { t->psi = cand; break; }
    }
    if (!t->psi) throw std::runtime_error("no 2n-th root of unity found");
    const u64 psi_inv = inv_mod(t->psi, p);
    std::vector<u64> pw(n), pwi(n);
    pw[0] = pwi[0] = 1;
    for (u32 i = 1; i < n; ++i) {
      pw[i] = mul_mod(pw[i - 1], t->psi, p);
      pwi[i] = mul_mod(pwi[i - 1], psi_inv, p);
    }
    t->fwd.resize(n); t->inv.resize(n); t->fwd_p.resize(n); t->inv_p.resize(n);
    for (u32 i = 0; i < n; ++i) {
      u32 r = bit_reverse(i, log_n);
      t->fwd[i] = pw[r];
      t->inv[i] = pwi[r];
      t->fwd_p[i] = shoup_pre(t->fwd[i], p);
      t->inv_p[i] = shoup_pre(t->inv[i], p);
    }
    t->n_inv = inv_mod(n, p);
    t->n_inv_p = shoup_pre(t->n_inv, p);
    return t;
  }

  std::shared_ptr<ConvPlan> plan(const u32* src, u32 k, const u32* dst, u32 m) {
    std::vector<u32> key(src, src + k);
    key.push_back(0xffffffffu);
    key.insert(key.end(), dst, dst + m);
    std::lock_guard<std::mutex> g(mu);
    auto it = plans.find(key);
    if (it != plans.end()) return it->second;
    auto pl = std::make_shared<ConvPlan>();
    for (u32 i = 0; i < k; ++i) pl->src_p.push_back(prime[src[i]]);
    for (u32 t = 0; t < m; ++t) pl->dst_p.push_back(prime[dst[t]]);
    pl->b_big = Big{1};
    for (u64 b : pl->src_p) big_mul_small(pl->b_big, b);
    for (u32 i = 0; i < k; ++i) {
      Big h{1};
      for (u32 j = 0; j < k; ++j) if (j != i) big_mul_small(h, pl->src_p[j]);
      pl->hat_big.push_back(h);
      const u64 bi = pl->src_p[i];
      const u64 hinv = inv_mod(big_mod_small(h, bi), bi);
      pl->hat_inv.push_back(hinv);
      pl->hat_inv_p.push_back(shoup_pre(hinv, bi));
      // floor(2^128 / b) = (floor(2^128-1)/b) since b does not divide 2^128
      u128 all = ~(u128)0;
      u128 w = all / bi;
      pl->w_hi.push_back((u64)(w >> 64));
      pl->w_lo.push_back((u64)w);
      for (u32 t = 0; t < m; ++t) pl->hat_mod.push_back(big_mod_small(h, pl->dst_p[t]));
    }
    for (u32 t = 0; t < m; ++t) pl->b_mod.push_back(big_mod_small(pl->b_big, pl->dst_p[t]));
    plans[key] = pl;
    return pl;
  }
};

namespace {

// ---- NTT kernels (rns_math.hpp:68-100) ------------------------------------
void ntt_forward(const NttTable& t, u64* a, u32 n) {
  const u64 p = t.p;
  u32 h = n;
  for (u32 m = 1; m < n; m <<= 1) {
    h >>= 1;
    for (u32 i = 0; i < m; ++i) {
      const u64 w = t.fwd[m + i], wp = t.fwd_p[m + i];
      u64* x = a + 2 * i * h;
      u64* y = x + h;
      for (u32 j = 0; j < h; ++j) {
        const u64 u = x[j];
        const u64 v = shoup_mul(y[j], w, wp, p);
        x[j] = add_mod(u, v, p);
        y[j] = sub_mod(u, v, p);
      }
    }
  }
}

void ntt_inverse(const NttTable& t, u64* a, u32 n) {
  const u64 p = t.p;
  u32 h = 1;
  for (u32 m = n; m > 1; m >>= 1) {
    const u32 half = m >> 1;
    for (u32 i = 0; i < half; ++i) {
      const u64 w = t.inv[half + i], wp = t.inv_p[half + i];
      u64* x = a + 2 * i * h;
      u64* y = x + h;
      for (u32 j = 0; j < h; ++j) {
        const u64 u = x[j], v = y[j];
        x[j] = add_mod(u, v, p);
        y[j] = shoup_mul(sub_mod(u, v, p), w, wp, p);
      }
    }
    h <<= 1;
  }
  for (u32 j = 0; j < n; ++j) a[j] = shoup_mul(a[j], t.n_inv, t.n_inv_p, p);
}

// ---- exact centred basis conversion ---------------------------------------
// Returns the number of near-tie fallbacks used for this coefficient (0/1).
inline int convert_coeff(const ConvPlan& pl, const u64* xs, size_t xstride, u64* out,
                         size_t ostride, u64* scratch) {
  const u32 k = (u32)pl.src_p.size();
  const u32 m = (u32)pl.dst_p.size();
  u128 F = 0;
  for (u32 i = 0; i < k; ++i) {
    const u64 xt = shoup_mul(xs[i * xstride], pl.hat_inv[i], pl.hat_inv_p[i], pl.src_p[i]);
    scratch[i] = xt;
    F += (u128)(xt * pl.w_hi[i]) + (u64)(((u128)xt * pl.w_lo[i]) >> 64);
  }
  const u128 Fh = F + ((u128)1 << 63);
  u64 v = (u64)(Fh >> 64);
  const u64 low = (u64)Fh;
  int fb = 0;
  if (low >= (u64)0 - 2ull * k) {
    // ambiguous: v or v + 1.  v+1 iff 2X >= (2v+1) B  (B odd: never equal)
    fb = 1;
    Big X{0};
    for (u32 i = 0; i < k; ++i) {
      Big term = pl.hat_big[i];
      big_mul_small(term, scratch[i]);
      big_add(X, term);
    }
    big_mul_small(X, 2);
    Big rhs = pl.b_big;
    big_mul_small(rhs, 2 * v + 1);
    if (big_cmp(X, rhs) >= 0) v += 1;
  }
  for (u32 t = 0; t < m; ++t) {
    const u64 d = pl.dst_p[t];
    u128 s = 0;
    for (u32 i = 0; i < k; ++i) s += (u128)scratch[i] * pl.hat_mod[i * m + t];
    const u64 sm = (u64)(s % d);
    const u64 vb = (u64)(((u128)v * pl.b_mod[t]) % d);
    out[t * ostride] = sub_mod(sm, vb, d);
  }
  return fb;
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
uint64_t orc_mix64(uint64_t x) { return mix64(x); }
uint64_t orc_row_key(uint64_t seed, uint64_t tag, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  return row_key(seed, tag, a, b, c, d);
}
void orc_fill_uniform(uint64_t rk, uint64_t p, uint64_t* out, uint32_t n) {
  const int sh = 64 - bitlen(p);
  for (u32 i = 0; i < n; ++i) out[i] = uniform_at(rk, i, p, sh);
}

orc_ctx* orc_create(uint32_t log_n, uint32_t chain, uint32_t lboot, uint64_t seed_input,
                    uint64_t seed_weight, uint64_t seed_key, int threads) {
  if (log_n < 3 || log_n > AEGIS_MAX_LOG_N || chain == 0 || chain > AEGIS_MAX_MAIN_PRIMES) {
    g_err = "orc_create: bad parameters";
    return nullptr;
  }
  auto* c = new orc_ctx;
  c->log_n = log_n;
  c->n = 1u << log_n;
  c->chain = chain;
  c->lboot = lboot;
  c->seed_input = seed_input;
  c->seed_weight = seed_weight;
  c->seed_key = seed_key;
  c->threads = threads > 0 ? threads : omp_get_max_threads();
  for (u32 i = 0; i < AEGIS_MAX_MAIN_PRIMES; ++i) c->prime.push_back(AEGIS_MAIN_PRIMES[i]);
  for (u32 i = 0; i < AEGIS_SPECIAL_PRIMES; ++i) c->prime.push_back(AEGIS_SPECIAL_PRIMES_LIST[i]);
  for (u64 p : c->prime) c->shift.push_back(64 - bitlen(p));
  c->tables.resize(c->prime.size());
  return c;
}
void orc_destroy(orc_ctx* c) { delete c; }
uint64_t orc_prime(const orc_ctx* c, uint32_t e) { return c->prime.at(e); }
uint64_t orc_psi(orc_ctx* c, uint32_t e) { return c->table(e).psi; }

int orc_ntt(orc_ctx* c, uint64_t* data, const uint32_t* ext_idx, uint32_t nlimbs, int inverse) {
  try {
    for (u32 k = 0; k < nlimbs; ++k) c->table(ext_idx[k]);
#pragma omp parallel for num_threads(c->threads) schedule(dynamic, 1)
    for (long k = 0; k < (long)nlimbs; ++k) {
      const NttTable& t = *c->tables[ext_idx[k]];
      if (inverse) ntt_inverse(t, data + (size_t)k * c->n, c->n);
      else ntt_forward(t, data + (size_t)k * c->n, c->n);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

uint64_t orc_galois(int offset, uint32_t n) {
  // rns_math.hpp:142-149: 5^offset mod 2n, offset taken mod n
  const u64 order = 2ull * n;
  long long ofs = offset % (long long)n;
  if (ofs < 0) ofs += n;
  u64 k = 1;
  for (long long i = 0; i < ofs; ++i) k = (k * 5) % order;
  return k;
}

int orc_automorphism_eval(orc_ctx* c, const uint64_t* in, uint64_t* out, uint32_t nlimbs, uint64_t k) {
  const u32 n = c->n, lg = c->log_n;
  const u64 mask = 2ull * n - 1;
  std::vector<u32> idx(n);
  for (u32 j = 0; j < n; ++j) {
    const u64 e = ((2ull * bit_reverse(j, lg) + 1) * k) & mask;  // odd exponent
    idx[j] = bit_reverse((u32)((e - 1) >> 1), lg);
  }
  for (u32 l = 0; l < nlimbs; ++l)
    for (u32 j = 0; j < n; ++j) out[(size_t)l * n + j] = in[(size_t)l * n + idx[j]];
  return 0;
}

int orc_ntt_prime(orc_ctx* c, uint64_t* data, uint64_t p, int inverse) {
  try {
    auto t = c->build_table(p);
    if (inverse) ntt_inverse(*t, data, c->n);
    else ntt_forward(*t, data, c->n);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int orc_automorphism_coeff(orc_ctx* c, const uint64_t* in, uint64_t* out, uint64_t p, uint64_t k) {
  // rns_math.hpp:127-139
  const u32 n = c->n;
  std::fill(out, out + n, 0);
  for (u32 i = 0; i < n; ++i) {
    const u64 pos = ((u64)i * k) % (2ull * n);
    if (pos < n) out[pos] = add_mod(out[pos], in[i], p);
    else out[pos - n] = sub_mod(out[pos - n], in[i], p);
  }
  return 0;
}

int64_t orc_basis_convert(orc_ctx* c, const uint64_t* in, const uint32_t* src, uint32_t k,
                          uint64_t* out, const uint32_t* dst, uint32_t m) {
  auto pl = c->plan(src, k, dst, m);
  const u32 n = c->n;
  int64_t fb = 0;
#pragma omp parallel for num_threads(c->threads) reduction(+ : fb) schedule(static)
  for (long j = 0; j < (long)n; ++j) {
    u64 scratch[128];
    fb += convert_coeff(*pl, in + j, n, out + j, n, scratch);
  }
  return fb;
}

int orc_basis_convert_bigint(orc_ctx* c, const uint64_t* in, const uint32_t* src, uint32_t k,
                             uint64_t* out, const uint32_t* dst, uint32_t m) {
  auto pl = c->plan(src, k, dst, m);
  const u32 n = c->n;
  Big half = pl->b_big;  // (B-1)/2
  {
    u64 carry = 0;
    for (size_t i = half.size(); i-- > 0;) {
      u128 cur = ((u128)carry << 64) | half[i];
      half[i] = (u64)(cur / 2);
      carry = (u64)(cur % 2);
    }
    big_trim(half);
  }
#pragma omp parallel for num_threads(c->threads) schedule(static)
  for (long j = 0; j < (long)n; ++j) {
    Big X{0};
    for (u32 i = 0; i < k; ++i) {
      const u64 xt = mul_mod(in[(size_t)i * n + j], pl->hat_inv[i], pl->src_p[i]);
      Big term = pl->hat_big[i];
      big_mul_small(term, xt);
      big_add(X, term);
    }
    while (big_cmp(X, pl->b_big) >= 0) big_sub(X, pl->b_big);  // X mod B
    const bool neg = big_cmp(X, half) > 0;                      // centred: x - B
    for (u32 t = 0; t < m; ++t) {
      const u64 d = pl->dst_p[t];
      u64 r = big_mod_small(X, d);
      if (neg) r = sub_mod(r, pl->b_mod[t], d);
      out[(size_t)t * n + j] = r;
    }
  }
  return 0;
}

}  // extern "C"

// ===========================================================================
// HE operators.  Ciphertext lane layout: [comp][limb][N], limb i <-> q_i.
// ===========================================================================
namespace {

struct Ctx {
  orc_ctx* c;
  u32 n;
  u64 p(u32 e) const { return c->prime[e]; }
};

u32 dnum_of(u32 level) { return (level + AEGIS_SPECIAL_PRIMES - 1) / AEGIS_SPECIAL_PRIMES; }

// Key material for (key_id, digit, comp, ext) -- DESIGN.md §2.3 tag 3.
std::shared_ptr<std::vector<u64>> key_limb(orc_ctx* c, u64 key_id, u32 digit, u32 comp, u32 e) {
  std::vector<u64> k{key_id, digit, comp, e};
  {
    std::lock_guard<std::mutex> g(c->mu);
    auto it = c->key_cache.find(k);
    if (it != c->key_cache.end()) return it->second;
  }
  auto v = std::make_shared<std::vector<u64>>(c->n);
  const u64 rk = row_key(c->seed_key, 3, key_id, digit, comp, e);
  const int sh = c->shift[e];
  for (u32 i = 0; i < c->n; ++i) (*v)[i] = uniform_at(rk, i, c->prime[e], sh);
  std::lock_guard<std::mutex> g(c->mu);
  c->key_cache[k] = v;
  return v;
}

// Hybrid key switch (poly_ir.hpp:219-298).  d: l limbs (NTT).
void keyswitch(orc_ctx* c, const u64* d, u32 l, u64 key_id, u64* out0, u64* out1) {
  const u32 n = c->n;
  const u32 K = AEGIS_SPECIAL_PRIMES;
  const u32 ext = l + K;
  const u32 dn = dnum_of(l);
  std::vector<u32> eidx(ext);
  for (u32 i = 0; i < l; ++i) eidx[i] = i;
  for (u32 k = 0; k < K; ++k) eidx[l + k] = kSpecialBase + k;
  for (u32 e : eidx) c->table(e);
  // 1. Intt
  std::vector<u64> dc(d, d + (size_t)l * n);
  for (u32 i = 0; i < l; ++i) ntt_inverse(*c->tables[i], dc.data() + (size_t)i * n, n);
  // 2-3. ModUp per digit + KeyMul accumulation
  std::vector<u64> acc0((size_t)ext * n, 0), acc1((size_t)ext * n, 0);
  std::vector<u64> tmp((size_t)ext * n);
  for (u32 j = 0; j < dn; ++j) {
    const u32 lo = j * K, hi = std::min(l, lo + K);
    std::vector<u32> src, dst;
    for (u32 i = lo; i < hi; ++i) src.push_back(i);
    std::vector<u32> dst_pos;
    for (u32 t = 0; t < ext; ++t)
      if (t < lo || t >= hi) { dst.push_back(eidx[t]); dst_pos.push_back(t); }
    auto pl = c->plan(src.data(), (u32)src.size(), dst.data(), (u32)dst.size());
    std::vector<u64> conv((size_t)dst.size() * n);
    u64 scratch[16];
    for (u32 x = 0; x < n; ++x)
      convert_coeff(*pl, dc.data() + (size_t)lo * n + x, n, conv.data() + x, n, scratch);
    for (u32 q = 0; q < dst.size(); ++q) {
      ntt_forward(*c->tables[dst[q]], conv.data() + (size_t)q * n, n);
      std::copy(conv.begin() + (size_t)q * n, conv.begin() + (size_t)(q + 1) * n,
                tmp.begin() + (size_t)dst_pos[q] * n);
    }
    for (u32 t = lo; t < hi; ++t)
      std::copy(d + (size_t)t * n, d + (size_t)(t + 1) * n, tmp.begin() + (size_t)t * n);
    for (u32 t = 0; t < ext; ++t) {
      const u64 p = c->prime[eidx[t]];
      auto k0 = key_limb(c, key_id, j, 0, eidx[t]);
      auto k1 = key_limb(c, key_id, j, 1, eidx[t]);
      u64* a0 = acc0.data() + (size_t)t * n;
      u64* a1 = acc1.data() + (size_t)t * n;
      const u64* e = tmp.data() + (size_t)t * n;
      for (u32 x = 0; x < n; ++x) {
        a0[x] = add_mod(a0[x], mul_mod(e[x], (*k0)[x], p), p);
        a1[x] = add_mod(a1[x], mul_mod(e[x], (*k1)[x], p), p);
      }
    }
  }
  // 4. ModDown: out_i = (acc_i - NTT_i([INTT(acc_P)]_P mod q_i)) * P^{-1} mod q_i
  std::vector<u32> psrc(K), qdst(l);
  for (u32 k = 0; k < K; ++k) psrc[k] = kSpecialBase + k;
  for (u32 i = 0; i < l; ++i) qdst[i] = i;
  auto pl = c->plan(psrc.data(), K, qdst.data(), l);
  for (int comp = 0; comp < 2; ++comp) {
    std::vector<u64>& acc = comp ? acc1 : acc0;
    u64* out = comp ? out1 : out0;
    std::vector<u64> pc(acc.begin() + (size_t)l * n, acc.end());
    for (u32 k = 0; k < K; ++k) ntt_inverse(*c->tables[psrc[k]], pc.data() + (size_t)k * n, n);
    std::vector<u64> conv((size_t)l * n);
    u64 scratch[16];
    for (u32 x = 0; x < n; ++x) convert_coeff(*pl, pc.data() + x, n, conv.data() + x, n, scratch);
    for (u32 i = 0; i < l; ++i) {
      const u64 q = c->prime[i];
      u64 pinv = 1;
      for (u32 k = 0; k < K; ++k) pinv = mul_mod(pinv, c->prime[psrc[k]] % q, q);
      pinv = inv_mod(pinv, q);
      ntt_forward(*c->tables[i], conv.data() + (size_t)i * n, n);
      for (u32 x = 0; x < n; ++x)
        out[(size_t)i * n + x] =
            mul_mod(sub_mod(acc[(size_t)i * n + x], conv[(size_t)i * n + x], q), pinv, q);
    }
  }
}

void automorph_eval_lane(orc_ctx* c, const u64* in, u64* out, u32 limbs, u64 k) {
  orc_automorphism_eval(c, in, out, limbs, k);
}

// Rot (he_ir.hpp:224-241 op; poly_ir.hpp:239-251 + key 1000+r :300-305)
void rotate(orc_ctx* c, const u64* ct, u32 l, int offset, u64* out) {
  const u32 n = c->n;
  const size_t cs = (size_t)l * n;
  const u64 k = orc_galois(offset, n);
  std::vector<u64> a(2 * cs);
  automorph_eval_lane(c, ct, a.data(), l, k);
  automorph_eval_lane(c, ct + cs, a.data() + cs, l, k);
  std::vector<u64> k0(cs), k1(cs);
  keyswitch(c, a.data() + cs, l, 1000u + (u64)offset, k0.data(), k1.data());
  for (u32 i = 0; i < l; ++i) {
    const u64 q = c->prime[i];
    for (u32 x = 0; x < n; ++x) {
      const size_t o = (size_t)i * n + x;
      out[o] = add_mod(a[o], k0[o], q);
      out[cs + o] = k1[o];
    }
  }
}

// Relin (he_ir.hpp:275-284; key 0): (d0,d1,d2) -> (d0+k0, d1+k1)
void relin(orc_ctx* c, const u64* ct3, u32 l, size_t cstride, u64* out, size_t ostride) {
  const u32 n = c->n;
  const size_t cs = (size_t)l * n;
  std::vector<u64> k0(cs), k1(cs);
  keyswitch(c, ct3 + 2 * cstride, l, 0, k0.data(), k1.data());
  for (u32 i = 0; i < l; ++i) {
    const u64 q = c->prime[i];
    for (u32 x = 0; x < n; ++x) {
      const size_t o = (size_t)i * n + x;
      out[o] = add_mod(ct3[o], k0[o], q);
      out[ostride + o] = add_mod(ct3[cstride + o], k1[o], q);
    }
  }
}

// Rescale (poly_ir.hpp:341-354, div_round rns_math.hpp:196-202):
// out_i = (x_i - NTT_i([x_{l-1}]_{q_{l-1}} centred mod q_i)) * q_{l-1}^{-1}
void rescale_poly(orc_ctx* c, const u64* x, u32 l, u64* out) {
  const u32 n = c->n;
  const u64 ql = c->prime[l - 1];
  std::vector<u64> last(x + (size_t)(l - 1) * n, x + (size_t)l * n);
  ntt_inverse(c->table(l - 1), last.data(), n);
  std::vector<u64> r(n);
  for (u32 i = 0; i + 1 < l; ++i) {
    const u64 q = c->prime[i];
    const u64 qlm = ql % q;
    const u64 inv = inv_mod(ql % q, q);
    for (u32 j = 0; j < n; ++j) {
      const u64 v = last[j];
      r[j] = v > (ql - 1) / 2 ? sub_mod(v % q, qlm, q) : v % q;  // centred lift mod q_i
    }
    ntt_forward(c->table(i), r.data(), n);
    for (u32 j = 0; j < n; ++j)
      out[(size_t)i * n + j] = mul_mod(sub_mod(x[(size_t)i * n + j], r[j], q), inv, q);
  }
}

// Boot reset (poly_ir.hpp:355-368): value-preserving lift from
// level l to out_level: limbs < min(l, out) copied, limbs >= l converted from
// the exact centred lift over Q_l.
void boot_poly(orc_ctx* c, const u64* x, u32 l, u32 out_level, u64* out) {
  const u32 n = c->n;
  const u32 keep = std::min(l, out_level);
  std::copy(x, x + (size_t)keep * n, out);
  if (out_level <= l) return;
  std::vector<u64> xc(x, x + (size_t)l * n);
  for (u32 i = 0; i < l; ++i) ntt_inverse(c->table(i), xc.data() + (size_t)i * n, n);
  std::vector<u32> src(l), dst;
  for (u32 i = 0; i < l; ++i) src[i] = i;
  for (u32 i = l; i < out_level; ++i) dst.push_back(i);
  auto pl = c->plan(src.data(), l, dst.data(), (u32)dst.size());
  std::vector<u64> scratch(l);
  for (u32 j = 0; j < n; ++j)
    convert_coeff(*pl, xc.data() + j, n, out + (size_t)l * n + j, n, scratch.data());
  for (u32 i = l; i < out_level; ++i) ntt_forward(c->table(i), out + (size_t)i * n, n);
}

}  // namespace

extern "C" {

int orc_keyswitch(orc_ctx* c, const uint64_t* d, uint32_t level, uint64_t key_id,
                  uint64_t* out0, uint64_t* out1) {
  try {
    keyswitch(c, d, level, key_id, out0, out1);
    return 0;
  } catch (const std::exception& e) { g_err = e.what(); return -1; }
}
int orc_rotate(orc_ctx* c, const uint64_t* ct, uint32_t level, int offset, uint64_t* out) {
  try { rotate(c, ct, level, offset, out); return 0; }
  catch (const std::exception& e) { g_err = e.what(); return -1; }
}
int orc_relin(orc_ctx* c, const uint64_t* ct3, uint32_t level, uint64_t* out2) {
  try {
    const size_t cs = (size_t)level * c->n;
    relin(c, ct3, level, cs, out2, cs);
    return 0;
  } catch (const std::exception& e) { g_err = e.what(); return -1; }
}
int orc_rescale(orc_ctx* c, const uint64_t* ct, uint32_t level, uint64_t* out) {
  try {
    const size_t ci = (size_t)level * c->n, co = (size_t)(level - 1) * c->n;
    rescale_poly(c, ct, level, out);
    rescale_poly(c, ct + ci, level, out + co);
    return 0;
  } catch (const std::exception& e) { g_err = e.what(); return -1; }
}
int orc_boot_reset(orc_ctx* c, const uint64_t* ct, uint32_t level, uint32_t out_level, uint64_t* out) {
  try {
    const size_t ci = (size_t)level * c->n, co = (size_t)out_level * c->n;
    boot_poly(c, ct, level, out_level, out);
    boot_poly(c, ct + ci, level, out_level, out + co);
    return 0;
  } catch (const std::exception& e) { g_err = e.what(); return -1; }
}
int orc_cmult(orc_ctx* c, const uint64_t* a, const uint64_t* b, uint32_t level, uint64_t* out3) {
  const u32 n = c->n;
  const size_t cs = (size_t)level * n;
  for (u32 i = 0; i < level; ++i) {
    const u64 q = c->prime[i];
    for (u32 x = 0; x < n; ++x) {
      const size_t o = (size_t)i * n + x;
      const u64 a0 = a[o], a1 = a[cs + o], b0 = b[o], b1 = b[cs + o];
      out3[o] = mul_mod(a0, b0, q);
      out3[cs + o] = add_mod(mul_mod(a0, b1, q), mul_mod(a1, b0, q), q);
      out3[2 * cs + o] = mul_mod(a1, b1, q);
    }
  }
  return 0;
}
void orc_key_limb(orc_ctx* c, uint64_t key_id, uint32_t digit, uint32_t comp, uint32_t e, uint64_t* out) {
  auto v = key_limb(c, key_id, digit, comp, e);
  std::copy(v->begin(), v->end(), out);
}
void orc_weight_limb(orc_ctx* c, uint32_t bundle, uint32_t lane, uint32_t limb, uint64_t* out) {
  const u64 rk = row_key(c->seed_weight, 2, bundle, lane, 0, limb);
  for (u32 i = 0; i < c->n; ++i) out[i] = uniform_at(rk, i, c->prime[limb], c->shift[limb]);
}
void orc_input_limb(orc_ctx* c, uint32_t bundle, uint32_t lane, uint32_t comp, uint32_t limb, uint64_t* out) {
  const u64 rk = row_key(c->seed_input, 1, bundle, lane, comp, limb);
  for (u32 i = 0; i < c->n; ++i) out[i] = uniform_at(rk, i, c->prime[limb], c->shift[limb]);
}

uint64_t orc_hash_bundle_data(const uint64_t* data, uint32_t lanes, uint32_t comps_stride,
                              uint32_t comps, uint32_t level_stride, uint32_t level, uint32_t n) {
  // H = sum over dense positions of mix64(value + pos * GOLD)
  u64 h = 0;
  for (u32 ln = 0; ln < lanes; ++ln)
    for (u32 cp = 0; cp < comps; ++cp)
      for (u32 lb = 0; lb < level; ++lb) {
        const u64* src = data + (((size_t)ln * comps_stride + cp) * level_stride + lb) * n;
        const u64 base = (((u64)ln * comps + cp) * level + lb) * n;
        for (u32 x = 0; x < n; ++x) h += mix64(src[x] + (base + x) * kGold);
      }
  return h;
}

}  // extern "C"

// ===========================================================================
// Graph executor (SPEC.md:407-415 exec_sequential over the HE-op IR).
// ===========================================================================
namespace {

enum OpKind { kEncode = 0, kPAdd, kCAdd, kPMult, kCMult, kRot, kRelin, kRescale, kBoot };

struct Slice { u32 b, lane, count; };
struct GOp {
  u32 id, kind;
  int rot;
  Slice out;
  bool acc, aligned;
  u64 work;
  u32 use_level;
  std::vector<Slice> ins;
};
// Zero-initialised bundle storage backed by an anonymous mapping: pages are
// committed only when written, so a lane-subset run (orc_run_graph_tg) holds
// just the lanes it computes even though lane addressing stays dense.
struct LazyBuf {
  u64* p = nullptr;
  size_t bytes = 0;
  LazyBuf() = default;
  LazyBuf(const LazyBuf&) = delete;
  LazyBuf& operator=(const LazyBuf&) = delete;
  LazyBuf(LazyBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  ~LazyBuf() { release(); }
  void assign(size_t words) {
    release();
    if (!words) return;
    bytes = words * sizeof(u64);
    void* m = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
    if (m == MAP_FAILED) throw std::runtime_error("oracle: bundle mapping failed");
    p = (u64*)m;
  }
  void release() {
    if (p) munmap(p, bytes);
    p = nullptr;
    bytes = 0;
  }
  u64* data() { return p; }
};

struct GBundle {
  u32 id, lanes, level, comps, chunk = 0;
  LazyBuf data;  // [lane][comps_alloc][level][N]
  u32 comps_alloc = 0;
  u32 cur_comps = 0;
  bool live = false;
};

struct Graph {
  std::vector<GBundle> b;
  std::vector<GOp> ops;
  std::vector<u32> inputs;
};

Graph parse(const char* path) {
  std::ifstream f(path);
  if (!f) throw std::runtime_error(std::string("cannot open graph ") + path);
  Graph g;
  std::string line;
  while (std::getline(f, line)) {
    if (line.empty() || line[0] == '#') continue;
    std::istringstream s(line);
    std::string t;
    s >> t;
    if (t == "inputs") {
      u32 v;
      while (s >> v) g.inputs.push_back(v);
    } else if (t == "B") {
      GBundle bb;
      u32 cls, chunk, rep, app;
      s >> bb.id >> bb.lanes >> bb.level >> bb.comps >> cls >> chunk >> rep >> app;
      bb.chunk = chunk;
      if (bb.id != g.b.size()) throw std::runtime_error("bundle ids not dense");
      g.b.push_back(std::move(bb));
    } else if (t == "O") {
      GOp o;
      int acc, al, phase;
      u32 app, agg;
      size_t nin;
      s >> o.id >> o.kind >> o.rot >> o.out.b >> o.out.lane >> o.out.count >> acc >> al >> phase >>
          o.work >> o.use_level >> app >> agg >> nin;
      o.acc = acc != 0;
      o.aligned = al != 0;
      for (size_t i = 0; i < nin; ++i) {
        Slice sl;
        s >> sl.b >> sl.lane >> sl.count;
        o.ins.push_back(sl);
      }
      g.ops.push_back(std::move(o));
    }
  }
  return g;
}

// lane of operand slice `in` feeding output lane l of an op with n out lanes
// (he_ir.hpp:200-222 emit_per_lane rule)
inline u32 map_lane(const Slice& in, u32 l, u32 n) {
  return in.lane + (in.count == n ? l : l % in.count);
}

struct Exec {
  orc_ctx* c;
  Graph g;
  u32 n;
  std::vector<int64_t> last_use;
  uint64_t* hashes;
  uint64_t nhashes;
  // Lane-subset mode (orc_run_graph_tg): compute and hash only the lanes of
  // token group tg_sel.  Token-coherent placement (placement.hpp:175-182,
  // PAPER.md:406-421) restated independently of the product: a graph input's
  // lanes are token-major (lane / (lanes / tg_total)); a PCMM output lane
  // lane(t, o) belongs to t; every other output lane inherits the group of the
  // operand lane it reads (emit_per_lane, he_ir.hpp:200-222).
  u32 tg_total = 1;
  int tg_sel = -1;
  std::vector<std::vector<int32_t>> tag;  // [bundle][lane]

  bool owns(u32 b, u32 lane) const { return tg_sel < 0 || tag[b][lane] == tg_sel; }
  void tag_lanes() {
    tag.assign(g.b.size(), {});
    for (auto& b : g.b) tag[b.id].assign(b.lanes, -1);
    for (u32 id : g.inputs) {
      const u32 lanes = g.b[id].lanes;
      if (lanes % tg_total) throw std::logic_error("graph input lanes not a multiple of token groups");
      for (u32 l = 0; l < lanes; ++l) tag[id][l] = (int32_t)(l / (lanes / tg_total));
    }
    auto put = [&](u32 b, u32 lane, int32_t t) {
      if (tag[b][lane] >= 0 && tag[b][lane] != t) throw std::logic_error("lane written by two token groups");
      tag[b][lane] = t;
    };
    for (const GOp& o : g.ops) {
      if (o.kind == kEncode) continue;
      const u32 nl = o.out.count;
      if (o.kind == kPMult) {
        const Pcmm s = pcmm(o);
        for (u32 t = 0; t < s.tg; ++t)
          for (u32 oo = 0; oo < s.c_out; ++oo) put(o.out.b, o.out.lane + s.lane(t, oo), (int32_t)t);
        continue;
      }
      for (u32 l = 0; l < nl; ++l) {
        const int32_t t = tag[o.ins[0].b][map_lane(o.ins[0], l, nl)];
        if (t < 0) throw std::logic_error("op reads an untagged lane");
        for (size_t k = 1; k < o.ins.size(); ++k)
          if (tag[o.ins[k].b][map_lane(o.ins[k], l, nl)] != t)
            throw std::invalid_argument("op " + std::to_string(o.id) + " couples token groups: no lane-subset run");
        put(o.out.b, o.out.lane + l, t);
      }
    }
  }
  struct Pcmm {
    u32 tg, c_in, c_out, S, c_sub, chunk;
    u32 lane(u32 t, u32 oo) const { return S == 1 ? t * c_out + oo : (oo / c_sub) * chunk + t * c_sub + oo % c_sub; }
  };
  Pcmm pcmm(const GOp& o) const {
    const u64 in_l = o.ins[0].count, out_l = o.out.count, w_l = o.ins[1].count;
    u64 tg = 1;
    while (tg * tg * w_l < in_l * out_l) ++tg;
    if (tg * tg * w_l != in_l * out_l || in_l % tg || out_l % tg)
      throw std::logic_error("PMult lane shapes inconsistent");
    Pcmm s;
    s.tg = (u32)tg;
    s.c_in = (u32)(in_l / tg);
    s.c_out = (u32)(out_l / tg);
    if ((u64)s.c_in * s.c_out != w_l) throw std::logic_error("PMult weight lanes inconsistent");
    s.chunk = g.b[o.out.b].chunk;
    s.S = (s.chunk == 0 || s.chunk >= out_l) ? 1 : (u32)(out_l / s.chunk);
    if (s.c_out % s.S) throw std::logic_error("PMult sub-tensor split inconsistent");
    s.c_sub = s.c_out / s.S;
    return s;
  }
  // keys are regenerated on demand; keep the cache bounded at production size
  void trim_keys() {
    std::lock_guard<std::mutex> lk(c->mu);
    if (c->key_cache.size() * (size_t)n * 8 > ((size_t)6 << 30)) c->key_cache.clear();
  }

  u64* lane_ptr(GBundle& b, u32 lane, u32 comp = 0) {
    return b.data.data() + ((size_t)lane * b.comps_alloc + comp) * b.level * n;
  }
  void ensure(GBundle& b, u32 comps) {
    if (b.live) return;
    b.comps_alloc = std::max(b.comps, comps);
    b.data.assign((size_t)b.lanes * b.comps_alloc * b.level * n);
    b.live = true;
    b.cur_comps = b.comps_alloc;
  }
  void materialize_input(GBundle& b) {
    ensure(b, 2);
#pragma omp parallel for collapse(2) num_threads(c->threads)
    for (long ln = 0; ln < (long)b.lanes; ++ln)
      for (long cp = 0; cp < 2; ++cp)
        for (u32 lb = 0; lb < b.level && owns(b.id, (u32)ln); ++lb)
          orc_input_limb(c, b.id, (u32)ln, (u32)cp, lb, lane_ptr(b, (u32)ln, (u32)cp) + (size_t)lb * n);
  }
  void finish(GBundle& b) {
    if (!b.live) return;
    if (b.id < nhashes) {
      // DESIGN.md §2.4 over the owned lanes only (all lanes when tg_sel < 0)
      u64 h = 0;
      for (u32 ln = 0; ln < b.lanes; ++ln) {
        if (!owns(b.id, ln)) continue;
        for (u32 cp = 0; cp < b.cur_comps; ++cp)
          for (u32 lb = 0; lb < b.level; ++lb) {
            const u64* src = lane_ptr(b, ln, cp) + (size_t)lb * n;
            const u64 base = (((u64)ln * b.cur_comps + cp) * b.level + lb) * n;
            for (u32 x = 0; x < n; ++x) h += mix64(src[x] + (base + x) * kGold);
          }
      }
      hashes[b.id] = h;
    }
    b.data.release();
    b.live = false;
  }

  void run(int64_t max_ops) {
    if (tg_sel >= 0) tag_lanes();
    last_use.assign(g.b.size(), -1);
    for (size_t i = 0; i < g.ops.size(); ++i) {
      last_use[g.ops[i].out.b] = (int64_t)i;
      for (auto& s : g.ops[i].ins) last_use[s.b] = (int64_t)i;
    }
    for (u32 id : g.inputs) materialize_input(g.b[id]);
    const int64_t nops = max_ops < 0 ? (int64_t)g.ops.size() : std::min<int64_t>(max_ops, g.ops.size());
    for (int64_t i = 0; i < nops; ++i) {
      exec(g.ops[i]);
      const GOp& o = g.ops[i];
      std::vector<u32> touched{o.out.b};
      for (auto& s : o.ins) touched.push_back(s.b);
      for (u32 b : touched)
        if (last_use[b] == i && i + 1 < (int64_t)g.ops.size()) finish(g.b[b]);
    }
    for (auto& b : g.b) finish(b);
  }

  void exec(const GOp& o) {
    switch (o.kind) {
      case kEncode: return;  // weights are generated where consumed (kGenerate)
      case kPMult: return pmult(o);
      case kRot: return rot(o);
      case kCMult: return cmult(o);
      case kRelin: return relin_op(o);
      case kRescale: return rescale_op(o);
      case kCAdd: return cadd(o, false);
      case kPAdd: return cadd(o, true);
      case kBoot: return boot(o);
      default: throw std::logic_error("unknown op kind");
    }
  }

  void rot(const GOp& o) {
    GBundle& in = g.b[o.ins[0].b];
    GBundle& out = g.b[o.out.b];
    ensure(out, 2);
    const u32 L = o.use_level, nl = o.out.count;
    // pre-generate key limbs (shared by all lanes)
    trim_keys();
    for (u32 j = 0; j < dnum_of(L); ++j)
      for (u32 cp = 0; cp < 2; ++cp)
        for (u32 e = 0; e < L + AEGIS_SPECIAL_PRIMES; ++e)
          key_limb(c, 1000u + (u64)o.rot, j, cp, e < L ? e : kSpecialBase + (e - L));
#pragma omp parallel for num_threads(c->threads) schedule(dynamic, 1)
    for (long l = 0; l < (long)nl; ++l) {
      if (!owns(o.out.b, o.out.lane + (u32)l)) continue;
      const u32 il = map_lane(o.ins[0], (u32)l, nl);
      std::vector<u64> src(2 * (size_t)L * n), dst(2 * (size_t)L * n);
      for (u32 cp = 0; cp < 2; ++cp)
        std::copy(lane_ptr(in, il, cp), lane_ptr(in, il, cp) + (size_t)L * n, src.begin() + cp * (size_t)L * n);
      rotate(c, src.data(), L, o.rot, dst.data());
      for (u32 cp = 0; cp < 2; ++cp)
        std::copy(dst.begin() + cp * (size_t)L * n, dst.begin() + (cp + 1) * (size_t)L * n,
                  lane_ptr(out, o.out.lane + (u32)l, cp));
    }
    out.cur_comps = 2;
  }

  void relin_op(const GOp& o) {
    GBundle& b = g.b[o.out.b];
    const u32 L = o.use_level, nl = o.out.count;
    trim_keys();
    for (u32 j = 0; j < dnum_of(L); ++j)
      for (u32 cp = 0; cp < 2; ++cp)
        for (u32 e = 0; e < L + AEGIS_SPECIAL_PRIMES; ++e)
          key_limb(c, 0, j, cp, e < L ? e : kSpecialBase + (e - L));
    const size_t cstride = (size_t)b.level * n;
#pragma omp parallel for num_threads(c->threads) schedule(dynamic, 1)
    for (long l = 0; l < (long)nl; ++l) {
      if (!owns(o.out.b, o.out.lane + (u32)l)) continue;
      u64* p = lane_ptr(b, o.out.lane + (u32)l);
      std::vector<u64> res(2 * cstride);
      relin(c, p, L, cstride, res.data(), cstride);
      std::copy(res.begin(), res.end(), p);
    }
    b.cur_comps = 2;
  }

  void cmult(const GOp& o) {
    GBundle& a = g.b[o.ins[0].b];
    GBundle& bb = g.b[o.ins[1].b];
    GBundle& out = g.b[o.out.b];
    ensure(out, 3);
    const u32 L = o.use_level, nl = o.out.count;
#pragma omp parallel for collapse(2) num_threads(c->threads)
    for (long l = 0; l < (long)nl; ++l)
      for (long i = 0; i < (long)L; ++i) {
        if (!owns(o.out.b, o.out.lane + (u32)l)) continue;
        const u32 la = map_lane(o.ins[0], (u32)l, nl), lb = map_lane(o.ins[1], (u32)l, nl);
        const u64 q = c->prime[i];
        const u64* a0 = lane_ptr(a, la, 0) + i * n; const u64* a1 = lane_ptr(a, la, 1) + i * n;
        const u64* b0 = lane_ptr(bb, lb, 0) + i * n; const u64* b1 = lane_ptr(bb, lb, 1) + i * n;
        u64* d0 = lane_ptr(out, o.out.lane + (u32)l, 0) + i * n;
        u64* d1 = lane_ptr(out, o.out.lane + (u32)l, 1) + i * n;
        u64* d2 = lane_ptr(out, o.out.lane + (u32)l, 2) + i * n;
        for (u32 x = 0; x < n; ++x) {
          const u64 x0 = a0[x], x1 = a1[x], y0 = b0[x], y1 = b1[x];
          d0[x] = mul_mod(x0, y0, q);
          d1[x] = (u64)((((u128)x0 * y1) + (u128)x1 * y0) % q);
          d2[x] = mul_mod(x1, y1, q);
        }
      }
    out.cur_comps = 3;
  }

  void rescale_op(const GOp& o) {
    GBundle& in = g.b[o.ins[0].b];
    GBundle& out = g.b[o.out.b];
    ensure(out, 2);
    const u32 L = o.use_level, nl = o.out.count;
#pragma omp parallel for collapse(2) num_threads(c->threads) schedule(dynamic, 1)
    for (long l = 0; l < (long)nl; ++l)
      for (long cp = 0; cp < 2; ++cp) {
        if (!owns(o.out.b, o.out.lane + (u32)l)) continue;
        const u32 il = map_lane(o.ins[0], (u32)l, nl);
        rescale_poly(c, lane_ptr(in, il, (u32)cp), L, lane_ptr(out, o.out.lane + (u32)l, (u32)cp));
      }
    out.cur_comps = 2;
  }

  void boot(const GOp& o) {
    GBundle& in = g.b[o.ins[0].b];
    GBundle& out = g.b[o.out.b];
    ensure(out, 2);
    const u32 L = o.use_level, nl = o.out.count;
#pragma omp parallel for collapse(2) num_threads(c->threads) schedule(dynamic, 1)
    for (long l = 0; l < (long)nl; ++l)
      for (long cp = 0; cp < 2; ++cp) {
        if (!owns(o.out.b, o.out.lane + (u32)l)) continue;
        const u32 il = map_lane(o.ins[0], (u32)l, nl);
        boot_poly(c, lane_ptr(in, il, (u32)cp), L, out.level, lane_ptr(out, o.out.lane + (u32)l, (u32)cp));
      }
    out.cur_comps = 2;
  }

  // CAdd / PAdd: out[l] = in0[m0(l)] + in1[m1(l)]  or, accumulating, out[l] += in0[m0(l)]
  void cadd(const GOp& o, bool plain) {
    GBundle& out = g.b[o.out.b];
    ensure(out, 2);
    const u32 L = o.use_level, nl = o.out.count;
    if (plain) throw std::logic_error("PAdd is not emitted by the reference lowering");
    const bool acc = o.acc;
    if (!acc && o.ins.size() != 2) throw std::logic_error("CAdd needs two operands");
#pragma omp parallel for collapse(3) num_threads(c->threads)
    for (long l = 0; l < (long)nl; ++l)
      for (long cp = 0; cp < 2; ++cp)
        for (long i = 0; i < (long)L; ++i) {
          if (!owns(o.out.b, o.out.lane + (u32)l)) continue;
          const u64 q = c->prime[i];
          u64* d = lane_ptr(out, o.out.lane + (u32)l, (u32)cp) + i * n;
          GBundle& a = g.b[o.ins[0].b];
          const u64* x = lane_ptr(a, map_lane(o.ins[0], (u32)l, nl), (u32)cp) + i * n;
          if (acc) {
            for (u32 t = 0; t < n; ++t) d[t] = add_mod(d[t], x[t], q);
          } else {
            GBundle& b = g.b[o.ins[1].b];
            const u64* y = lane_ptr(b, map_lane(o.ins[1], (u32)l, nl), (u32)cp) + i * n;
            for (u32 t = 0; t < n; ++t) d[t] = add_mod(x[t], y[t], q);
          }
        }
    out.cur_comps = 2;
  }

  // Bundled PCMM step (he_ir.hpp:360-371):
  //   acc[lane(t, o)] += sum_i X[t*c_in + i] * W[i*c_out + o]
  // where an accumulator of S = lanes / chunk_period sub-tensors (QKV: S = 3,
  // he_ir.hpp:338) is sub-tensor-major, token-major inside each sub-tensor:
  //   lane(t, o) = (o / c_sub) * chunk_period + t * c_sub + o % c_sub.
  void pmult(const GOp& o) {
    if (!o.acc || o.ins.size() != 2) throw std::logic_error("PMult form not supported");
    GBundle& acc = g.b[o.out.b];
    ensure(acc, 2);
    GBundle& X = g.b[o.ins[0].b];
    const u32 wb = o.ins[1].b;
    const Pcmm s = pcmm(o);
    const u32 c_in = s.c_in, c_out = s.c_out, tg = s.tg;
    const u32 L = o.use_level;
    auto acc_lane = [&](u32 t, u32 oo) { return s.lane(t, oo); };
#pragma omp parallel for collapse(2) num_threads(c->threads) schedule(dynamic, 1)
    for (long i = 0; i < (long)L; ++i)
      for (long oo = 0; oo < (long)c_out; ++oo) {
        const u64 q = c->prime[i];
        std::vector<u64> w((size_t)c_in * n);
        for (u32 ci = 0; ci < c_in; ++ci)
          orc_weight_limb(c, wb, ci * c_out + (u32)oo, (u32)i, w.data() + (size_t)ci * n);
        for (u32 t = 0; t < tg; ++t)
          for (u32 cp = 0; cp < 2 && (tg_sel < 0 || (int)t == tg_sel); ++cp) {
            u64* d = lane_ptr(acc, o.out.lane + acc_lane(t, (u32)oo), cp) + i * n;
            for (u32 x = 0; x < n; ++x) {
              u128 s = d[x];
              for (u32 ci = 0; ci < c_in; ++ci)
                s += (u128)lane_ptr(X, o.ins[0].lane + t * c_in + ci, cp)[i * n + x] * w[(size_t)ci * n + x];
              d[x] = (u64)(s % q);
            }
          }
      }
    acc.cur_comps = 2;
  }
};

}  // namespace

extern "C" int64_t orc_run_graph(orc_ctx* c, const char* path, int64_t max_ops, uint64_t* hashes,
                                 uint64_t nhashes) {
  return orc_run_graph_tg(c, path, max_ops, hashes, nhashes, 1, -1);
}

extern "C" int64_t orc_run_graph_tg(orc_ctx* c, const char* path, int64_t max_ops, uint64_t* hashes,
                                    uint64_t nhashes, uint32_t tg_total, int32_t tg_sel) {
  try {
    if (tg_total == 0 || tg_sel >= (int32_t)tg_total) throw std::invalid_argument("bad token-group selection");
    Exec ex{c, parse(path), c->n, {}, hashes, nhashes};
    ex.tg_total = tg_total;
    ex.tg_sel = tg_sel;
    if (hashes) std::fill(hashes, hashes + nhashes, 0);
    ex.run(max_ops);
    return (int64_t)ex.g.b.size();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

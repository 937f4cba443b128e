// context.cu -- device context, tables, keys, and the HE operators of libaegis.
//
// Host orchestration of the hot path.  Every operator is a short sequence of
// sm_100a kernels on the context's compute stream; no CPU arithmetic touches
// ciphertext data.  Reference anchors (proj/include/heplan/):
//   NTT tables       rns_math.hpp:46-63, 103-117
//   key switch       poly_ir.hpp:219-305 (Intt, Auto, ModUp, KeyMul, ModDown, Ntt)
//   rescale          poly_ir.hpp:341-354 + div_round rns_math.hpp:196-202
//   boot reset       poly_ir.hpp:355-368
//   pointwise ops    poly_ir.hpp:192-213
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "context.h"

namespace aegis {

namespace {

using u128h = unsigned __int128;

u64 h_mulmod(u64 a, u64 b, u64 p) { return (u64)(((u128h)a * b) % p); }
u64 h_powmod(u64 b, u64 e, u64 p) {
  u64 r = 1 % p;
  b %= p;
  while (e) {
    if (e & 1) r = h_mulmod(r, b, p);
    b = h_mulmod(b, b, p);
    e >>= 1;
  }
  return r;
}
u64 h_inv(u64 a, u64 p) { return h_powmod(a % p, p - 2, p); }
u64 h_shoup(u64 w, u64 p) { return (u64)(((u128h)w << 64) / p); }
u32 h_brev(u32 v, int bits) {
  u32 r = 0;
  for (int i = 0; i < bits; ++i, v >>= 1) r = (r << 1) | (v & 1);
  return r;
}

// multiword helpers for conversion plans
using Big = std::vector<u64>;
void big_mul(Big& a, u64 m) {
  u64 c = 0;
  for (auto& w : a) {
    u128h t = (u128h)w * m + c;
    w = (u64)t;
    c = (u64)(t >> 64);
  }
  if (c) a.push_back(c);
}
u64 big_mod(const Big& a, u64 p) {
  u128h r = 0;
  for (size_t i = a.size(); i-- > 0;) r = ((r << 64) | a[i]) % p;
  return (u64)r;
}

}  // namespace

Context::Context(const aegis_params& prm, int dev) {
  if (prm.log_n < 4 || prm.log_n > AEGIS_MAX_LOG_N)
    throw Error(AEGIS_EINVAL, "ring_degree must be a power of two in [2^4, 2^17]");
  if (prm.chain_length == 0 || prm.chain_length > AEGIS_MAX_MAIN_PRIMES)
    throw Error(AEGIS_EINVAL, "chain_length must be in [1, 60]");
  if (prm.special_primes != AEGIS_SPECIAL_PRIMES)
    throw Error(AEGIS_EINVAL, "special_prime_count must be 4");
  if (prm.bootstrap_level > prm.chain_length)
    throw Error(AEGIS_EINVAL, "bootstrap_level exceeds chain_length");  // ckks.hpp:45
  log_n = prm.log_n;
  n = 1u << log_n;
  chain = prm.chain_length;
  lboot = prm.bootstrap_level;
  seed_input = prm.seed_input;
  seed_weight = prm.seed_weight;
  seed_key = prm.seed_key;
  device = dev;
  AEGIS_CHECK_CUDA(cudaSetDevice(dev));
  AEGIS_CHECK_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  AEGIS_CHECK_CUDA(cudaStreamCreateWithFlags(&comm, cudaStreamNonBlocking));
  AEGIS_CHECK_CUDA(cudaDeviceGetDefaultMemPool(&pool_, dev));
  u64 thresh = ~0ull;  // keep freed blocks cached in the pool
  AEGIS_CHECK_CUDA(cudaMemPoolSetAttribute(pool_, cudaMemPoolAttrReleaseThreshold, &thresh));

  for (u32 i = 0; i < AEGIS_MAX_MAIN_PRIMES; ++i) primes_.push_back(AEGIS_MAIN_PRIMES[i]);
  for (u32 i = 0; i < AEGIS_SPECIAL_PRIMES; ++i) primes_.push_back(AEGIS_SPECIAL_PRIMES_LIST[i]);

  // ---- per-prime constants + twiddle tables (rns_math.hpp:46-63) ----
  std::vector<PrimeConst> pc(kNumExt);
  std::vector<PrimeTw> tw(kNumExt);
  std::vector<NttScale> sc(kNumExt);
  const size_t tab_words = (size_t)n * 2;  // ulonglong2 per entry
  // per prime: int fwd, int inv, f64 fwd, f64 inv
  AEGIS_CHECK_CUDA(cudaMalloc(&d_twiddles_, (size_t)kNumExt * 4 * tab_words * sizeof(u64)));
  std::vector<u64> hf(tab_words), hi(tab_words), pw(n), pwi(n);
  std::vector<double> ff(tab_words), fi(tab_words), fw(n), iw(n);
  AEGIS_CHECK_CUDA(cudaMalloc(&d_twd_, (size_t)kNumExt * 2 * n * sizeof(double)));
  const size_t blob_words = log_n == 16 ? (size_t)16 * kNttBlobTile : 0;
  std::vector<double> fblob(blob_words), iblob(blob_words);
  if (blob_words) AEGIS_CHECK_CUDA(cudaMalloc(&d_blob_, (size_t)kNumExt * 2 * blob_words * sizeof(double)));
  if (const char* impl = std::getenv("AEGIS_NTT_IMPL")) g_ntt_impl = std::string(impl) == "int" ? kNttInt : kNttF64;
  if (const char* v2 = std::getenv("AEGIS_NTT_V2")) g_ntt_v2 = std::string(v2) != "0";
  if (const char* cf = std::getenv("AEGIS_CONV_FUSED")) g_conv_fused = std::string(cf) != "0";
  if (const char* pd = std::getenv("AEGIS_PDL")) g_pdl = std::string(pd) != "0";
  if (const char* kf = std::getenv("AEGIS_KM_F64")) g_km_f64 = std::string(kf) != "0";
  if (const char* wsv = std::getenv("AEGIS_WS_SCALE")) ws_scale = std::max(0.001, std::atof(wsv));
  if (const char* ks = std::getenv("AEGIS_KM_SPLIT")) g_km_split = std::string(ks) != "0";

  for (u32 e = 0; e < kNumExt; ++e) {
    const u64 p = primes_[e];
    pc[e].p = p;
    pc[e].mu104 = (u64)(((u128h)1 << 104) / p);
    pc[e].shift = (u32)__builtin_clzll(p);
    pc[e].pad = 0;
    // psi: first g >= 2 whose g^((p-1)/2n) has order 2n (rns_math.hpp:103-111)
    const u64 order = 2ull * n;
    u64 psi = 0;
    for (u64 g = 2; g < p; ++g) {
      const u64 cand = h_powmod(g, (p - 1) / order, p);
      if (h_powmod(cand, n, p) == p - 1) { psi = cand; break; }
    }
    if (!psi) throw Error(AEGIS_EINVAL, "no 2n-th root of unity found");
    const u64 psi_inv = h_inv(psi, p);
    pw[0] = pwi[0] = 1;
    for (u32 i = 1; i < n; ++i) {
      pw[i] = h_mulmod(pw[i - 1], psi, p);
      pwi[i] = h_mulmod(pwi[i - 1], psi_inv, p);
    }
    for (u32 i = 0; i < n; ++i) {
      const u32 r = h_brev(i, (int)log_n);
      hf[2 * i] = pw[r];
      hf[2 * i + 1] = h_shoup(pw[r], p);
      hi[2 * i] = pwi[r];
      hi[2 * i + 1] = h_shoup(pwi[r], p);
      ff[2 * i] = (double)pw[r];
      ff[2 * i + 1] = (double)pw[r] / (double)p;
      fi[2 * i] = (double)pwi[r];
      fi[2 * i + 1] = (double)pwi[r] / (double)p;
      fw[i] = (double)pw[r];
      iw[i] = (double)pwi[r];
    }
    double* fwd_w = d_twd_ + (size_t)e * 2 * n;
    AEGIS_CHECK_CUDA(cudaMemcpy(fwd_w, fw.data(), (size_t)n * 8, cudaMemcpyHostToDevice));
    AEGIS_CHECK_CUDA(cudaMemcpy(fwd_w + n, iw.data(), (size_t)n * 8, cudaMemcpyHostToDevice));
    tw[e].fw = fwd_w;
    tw[e].iw = fwd_w + n;
    tw[e].fb = tw[e].ib = nullptr;
    if (blob_words) {
      ntt_build_blob(fw.data(), fblob.data());
      ntt_build_blob(iw.data(), iblob.data());
      double* bf = d_blob_ + (size_t)e * 2 * blob_words;
      AEGIS_CHECK_CUDA(cudaMemcpy(bf, fblob.data(), blob_words * 8, cudaMemcpyHostToDevice));
      AEGIS_CHECK_CUDA(cudaMemcpy(bf + blob_words, iblob.data(), blob_words * 8, cudaMemcpyHostToDevice));
      tw[e].fb = bf;
      tw[e].ib = bf + blob_words;
    }
    u64* fdev = d_twiddles_ + (size_t)e * 4 * tab_words;
    u64* idev = fdev + tab_words;
    u64* f64dev = idev + tab_words;
    u64* i64dev = f64dev + tab_words;
    AEGIS_CHECK_CUDA(cudaMemcpy(fdev, hf.data(), tab_words * 8, cudaMemcpyHostToDevice));
    AEGIS_CHECK_CUDA(cudaMemcpy(idev, hi.data(), tab_words * 8, cudaMemcpyHostToDevice));
    AEGIS_CHECK_CUDA(cudaMemcpy(f64dev, ff.data(), tab_words * 8, cudaMemcpyHostToDevice));
    AEGIS_CHECK_CUDA(cudaMemcpy(i64dev, fi.data(), tab_words * 8, cudaMemcpyHostToDevice));
    tw[e].fwd = reinterpret_cast<const ulonglong2*>(fdev);
    tw[e].inv = reinterpret_cast<const ulonglong2*>(idev);
    tw[e].fwd64 = reinterpret_cast<const double2*>(f64dev);
    tw[e].inv64 = reinterpret_cast<const double2*>(i64dev);
    tw[e].p = p;
    const u64 ninv = h_inv(n, p);
    sc[e].n_inv = ninv;
    sc[e].n_inv_p = h_shoup(ninv, p);
    sc[e].w1n = h_mulmod(pwi[h_brev(1, (int)log_n)], ninv, p);  // inv[1] * N^{-1}
    sc[e].w1n_p = h_shoup(sc[e].w1n, p);
    sc[e].mu64 = (u64)((~(u128h)0 >> 64) / p);  // floor((2^64 - 1) / p) == floor(2^64 / p)
    sc[e].pd = (double)p;
    sc[e].pinv = 1.0 / (double)p;
    sc[e].n_inv_d = (double)ninv;
    sc[e].n_inv_wp = (double)ninv / (double)p;
    sc[e].w1n_d = (double)sc[e].w1n;
    sc[e].w1n_wp = (double)sc[e].w1n / (double)p;
  }
  AEGIS_CHECK_CUDA(cudaMalloc(&d_pc, sizeof(PrimeConst) * kNumExt));
  AEGIS_CHECK_CUDA(cudaMalloc(&d_tw, sizeof(PrimeTw) * kNumExt));
  AEGIS_CHECK_CUDA(cudaMalloc(&d_scale, sizeof(NttScale) * kNumExt));
  AEGIS_CHECK_CUDA(cudaMemcpy(d_pc, pc.data(), sizeof(PrimeConst) * kNumExt, cudaMemcpyHostToDevice));
  AEGIS_CHECK_CUDA(cudaMemcpy(d_tw, tw.data(), sizeof(PrimeTw) * kNumExt, cudaMemcpyHostToDevice));
  AEGIS_CHECK_CUDA(cudaMemcpy(d_scale, sc.data(), sizeof(NttScale) * kNumExt, cudaMemcpyHostToDevice));
  std::vector<u32> ident(kNumExt);
  for (u32 i = 0; i < kNumExt; ++i) ident[i] = i;
  AEGIS_CHECK_CUDA(cudaMalloc(&d_ident, sizeof(u32) * kNumExt));
  AEGIS_CHECK_CUDA(cudaMemcpy(d_ident, ident.data(), sizeof(u32) * kNumExt, cudaMemcpyHostToDevice));
  std::vector<u32> kse(key_slots());
  for (u32 s = 0; s < key_slots(); ++s) kse[s] = s < chain ? s : kSpecialBase + (s - chain);
  AEGIS_CHECK_CUDA(cudaMalloc(&d_key_slot_ext_, sizeof(u32) * kse.size()));
  AEGIS_CHECK_CUDA(cudaMemcpy(d_key_slot_ext_, kse.data(), sizeof(u32) * kse.size(), cudaMemcpyHostToDevice));
}

Context::~Context() {
  cudaSetDevice(device);
  cudaStreamSynchronize(stream);
  for (auto& kv : keys_) cudaFree(kv.second);
  for (auto& kv : plans_) cudaFree(kv.second.dev);
  cudaFree(d_twiddles_);
  cudaFree(d_twd_);
  cudaFree(d_blob_);
  cudaFree(d_pc);
  cudaFree(d_tw);
  cudaFree(d_scale);
  cudaFree(d_ident);
  cudaFree(d_key_slot_ext_);
  arena_.reset();
  cudaStreamDestroy(stream);
  cudaStreamDestroy(comm);
}

u64* Context::alloc(size_t words) {
  void* p = nullptr;
  if (!words) words = 1;
  const size_t bytes = words * sizeof(u64);
  if (bytes >= kArenaMin) {
    if (!arena_) arena_.reset(new Arena(device));
    p = arena_->alloc(bytes);
    if (!p) {
      // idle pool blocks (small allocations) hold physical memory too
      cudaStreamSynchronize(stream);
      cudaMemPoolTrimTo(pool_, 0);
      p = arena_->alloc(bytes);
    }
    if (p) return static_cast<u64*>(p);
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    throw Error(AEGIS_EOOM, std::string("device allocation of ") + std::to_string(bytes) +
                                " bytes failed (arena mapped " + std::to_string(arena_->mapped() >> 20) +
                                " MiB, in use " + std::to_string(arena_->in_use() >> 20) + " MiB, largest free " +
                                std::to_string(arena_->largest_free() >> 20) + " MiB; bundles live " +
                                std::to_string(live_bytes >> 20) + " MiB, keys " + std::to_string(total_key_bytes() >> 20) +
                                " MiB, device free " + std::to_string(fr >> 20) + " of " + std::to_string(tot >> 20) +
                                " MiB)");
  }
  cudaError_t e = cudaMallocAsync(&p, bytes, stream);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    cudaStreamSynchronize(stream);
    cudaMemPoolTrimTo(pool_, 0);
    if (arena_) arena_->trim();
    e = cudaMallocAsync(&p, bytes, stream);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(e == cudaErrorMemoryAllocation ? AEGIS_EOOM : AEGIS_ECUDA,
                std::string("device allocation of ") + std::to_string(bytes) + " bytes failed: " + cudaGetErrorString(e));
  }
  return static_cast<u64*>(p);
}
void Context::release(void* p) {
  if (!p) return;
  if (arena_ && arena_->owns(p)) {
    arena_->free(p);  // reuse is ordered after this stream's pending work
    return;
  }
  cudaFreeAsync(p, stream);
}
void Context::trim() {
  cudaStreamSynchronize(stream);
  cudaMemPoolTrimTo(pool_, 0);
  if (arena_) arena_->trim();
}

Bundle* Context::new_bundle(u32 lanes, u32 comps, u32 level, bool zero) {
  auto* b = new Bundle;
  b->lanes = lanes;
  b->comps = comps;
  b->level = level;
  const size_t words = (size_t)lanes * comps * level * n;
  b->bytes = words * 8;
  try {
    b->ptr = alloc(words);
  } catch (...) {
    delete b;
    throw;
  }
  if (zero) AEGIS_CHECK_CUDA(cudaMemsetAsync(b->ptr, 0, b->bytes, stream));
  live_bytes += b->bytes;
  peak_bytes = std::max(peak_bytes, live_bytes);
  return b;
}
void Context::free_bundle(Bundle* b) {
  if (!b) return;
  release(b->ptr);
  live_bytes -= b->bytes;
  delete b;
}

const Plan& Context::plan(const std::vector<u32>& src, const std::vector<u32>& dst) {
  std::vector<u32> key(src);
  key.push_back(0xffffffffu);
  key.insert(key.end(), dst.begin(), dst.end());
  auto it = plans_.find(key);
  if (it != plans_.end()) return it->second;
  const u32 k = (u32)src.size(), m = (u32)dst.size();
  if (k == 0 || k > (u32)kMaxConv || m > (u32)kMaxConv) throw Error(AEGIS_EINVAL, "conversion basis too large");
  ConvPlanDev h;
  std::memset(&h, 0, sizeof(h));
  h.k = k;
  h.m = m;
  Big B{1};
  for (u32 i = 0; i < k; ++i) big_mul(B, prime(src[i]));
  if (B.size() > (size_t)kMaxBigWords) throw Error(AEGIS_EINVAL, "conversion modulus too wide");
  h.big_words = (u32)B.size();
  for (size_t w = 0; w < B.size(); ++w) h.b_big[w] = B[w];
  std::vector<u64> hm((size_t)k * m), hmp((size_t)k * m), hb((size_t)k * h.big_words, 0);
  for (u32 i = 0; i < k; ++i) {
    const u64 b = prime(src[i]);
    Big hat{1};
    for (u32 j = 0; j < k; ++j)
      if (j != i) big_mul(hat, prime(src[j]));
    for (size_t w = 0; w < hat.size() && w < h.big_words; ++w) hb[(size_t)i * h.big_words + w] = hat[w];
    h.src_p[i] = b;
    h.src_mu[i] = (u64)(((u128h)1 << 104) / b);
    const u64 hinv = h_inv(big_mod(hat, b), b);
    h.hat_inv[i] = hinv;
    h.hat_inv_p[i] = h_shoup(hinv, b);
    const u128h wq = (~(u128h)0) / b;  // floor(2^128 / b): b does not divide 2^128
    h.w_hi[i] = (u64)(wq >> 64);
    h.w_lo[i] = (u64)wq;
    for (u32 t = 0; t < m; ++t) {
      const u64 d = prime(dst[t]);
      const u64 v = big_mod(hat, d);
      hm[(size_t)i * m + t] = v;
      hmp[(size_t)i * m + t] = h_shoup(v, d);
    }
  }
  for (u32 t = 0; t < m; ++t) {
    const u64 d = prime(dst[t]);
    h.dst_p[t] = d;
    h.dst_mu[t] = (u64)(((u128h)1 << 104) / d);
    h.b_mod[t] = big_mod(B, d);
    h.dst_mu96[t] = (u64)(((u128h)1 << 96) / d);
  }
  Plan pl;
  pl.k = k;
  pl.m = m;
  const size_t extra = hm.size() + hmp.size() + hb.size();
  char* mem = nullptr;
  AEGIS_CHECK_CUDA(cudaMalloc(&mem, sizeof(ConvPlanDev) + extra * 8));
  pl.dev = reinterpret_cast<ConvPlanDev*>(mem);
  pl.tables = reinterpret_cast<u64*>(mem + sizeof(ConvPlanDev));
  AEGIS_CHECK_CUDA(cudaMemcpy(pl.dev, &h, sizeof(h), cudaMemcpyHostToDevice));
  AEGIS_CHECK_CUDA(cudaMemcpy(pl.tables, hm.data(), hm.size() * 8, cudaMemcpyHostToDevice));
  AEGIS_CHECK_CUDA(cudaMemcpy(pl.tables + hm.size(), hmp.data(), hmp.size() * 8, cudaMemcpyHostToDevice));
  if (!hb.empty())
    AEGIS_CHECK_CUDA(cudaMemcpy(pl.tables + hm.size() + hmp.size(), hb.data(), hb.size() * 8,
                                cudaMemcpyHostToDevice));
  return plans_.emplace(key, pl).first->second;
}

u64* Context::alloc_key() {
  u64* k = nullptr;
  const size_t words = key_bytes() / 8;
  cudaError_t e = cudaMalloc(&k, words * 8);
  if (e != cudaSuccess) {  // idle arena / pool memory may hold the space: release it and retry
    cudaGetLastError();
    trim();
    e = cudaMalloc(&k, words * 8);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(AEGIS_EOOM, "key allocation failed");
  }
  return k;
}

// Rotation key for offset r = key_id - 1000 is stored pre-permuted by the
// inverse automorphism: key'_r = auto_{k^-1}(key_r).  Then
//   KS(auto_k(c1)) = auto_k(ModDown(sum_j ModUp(c1)_j * key'_j))
// exactly (auto_k is a signed coefficient permutation; the centred lift and
// the rounding division commute with it), so the ModUp of c1 no longer
// depends on the offset and can be hoisted across rotations.
void Context::prepermute_key(u64 key_id, u64* k) {
  if (key_id < 500) return;
  const size_t words = key_bytes() / 8;
  const u64 gk = galois_of((int)((long long)key_id - 1000));
  const u64 ginv = h_powmod(gk, (u64)n - 1, 2ull * n);  // k^-1 mod 2N (the group has order N)
  u64* tmp = alloc(words);
  const u32 rows = key_digits() * 2 * key_slots();
  AEGIS_CHECK_CUDA(launch_automorphism(View{tmp, rows, 1, 1}, LaneMap{0, rows}, View{k, rows, 1, 1},
                                       LaneMap{0, rows}, rows, 1, 1, log_n, ginv, stream));
  count();
  AEGIS_CHECK_CUDA(cudaMemcpyAsync(k, tmp, words * 8, cudaMemcpyDeviceToDevice, stream));
  release(tmp);
}

void Context::generate_key(u64 key_id) {
  if (keys_.count(key_id)) return;
  u64* k = alloc_key();
  AEGIS_CHECK_CUDA(launch_fill_key(k, key_digits(), key_slots(), n, seed_key, key_id, d_key_slot_ext_, d_pc, stream));
  count();
  prepermute_key(key_id, k);
  keys_[key_id] = k;
}

// Caller-supplied key (SURVEY §8(b) aegis_keys_upload): [digit][comp][slot][N]
// canonical residues, slot s < chain -> q_s, else P_{s - chain}.  Digit j holds
// the key for the lift of limbs [4j, 4j+4) (key_switch, poly_ir.hpp:219-298,
// hybrid form).  Rotation keys are given in the standard (unpermuted) form.
void Context::upload_key(u64 key_id, const u64* host, size_t words, bool coeff_domain) {
  if (words != key_bytes() / 8)
    throw Error(AEGIS_EINVAL, "key upload: expected " + std::to_string(key_bytes() / 8) + " words, got " +
                                  std::to_string(words));
  auto it = keys_.find(key_id);
  if (it != keys_.end()) {
    AEGIS_CHECK_CUDA(cudaStreamSynchronize(stream));
    cudaFree(it->second);
    keys_.erase(it);
  }
  u64* k = alloc_key();
  AEGIS_CHECK_CUDA(cudaMemcpyAsync(k, host, words * 8, cudaMemcpyHostToDevice, stream));
  if (coeff_domain) {
    std::vector<u32> off(key_slots()), pr(key_slots());
    for (u32 s = 0; s < key_slots(); ++s) {
      off[s] = s;
      pr[s] = s < chain ? s : kSpecialBase + (s - chain);
    }
    ntt(k, (size_t)key_slots() * n, key_digits() * 2, off, pr, false);
  }
  prepermute_key(key_id, k);
  AEGIS_CHECK_CUDA(cudaStreamSynchronize(stream));  // the host buffer may be pageable / reused
  keys_[key_id] = k;
}

u64 Context::galois_of(int offset) const {  // 5^offset mod 2N (rns_math.hpp:142-149)
  const u64 order = 2ull * n;
  long long ofs = offset % (long long)n;
  if (ofs < 0) ofs += n;
  u64 gk = 1;
  for (long long i = 0; i < ofs; ++i) gk = (gk * 5) % order;
  return gk;
}
u64* Context::key_storage(u64 key_id, bool create) {
  auto it = keys_.find(key_id);
  if (it != keys_.end()) return it->second;
  if (!create) return nullptr;
  u64* k = alloc_key();
  keys_[key_id] = k;
  return k;
}

void Context::drop_key(u64 key_id) {
  auto it = keys_.find(key_id);
  if (it == keys_.end()) return;
  cudaStreamSynchronize(stream);
  cudaFree(it->second);
  keys_.erase(it);
}

u64 Context::chain_fingerprint() const {
  u64 h = mix64(log_n * kGold + chain);
  for (u32 i = 0; i < chain; ++i) h = mix64(h ^ (primes_[i] + (i + 1) * kGold));
  for (u32 i = 0; i < kAlpha; ++i) h = mix64(h ^ (primes_[kSpecialBase + i] + (i + 101) * kGold));
  return h;
}

const u64* Context::key(u64 key_id) {
  auto it = keys_.find(key_id);
  if (it == keys_.end()) generate_key(key_id);
  return keys_.at(key_id);
}

// ---------------------------------------------------------------------------
void Context::ntt(u64* base, size_t lane_stride, u32 nlanes, const std::vector<u32>& slot_off,
                  const std::vector<u32>& primes, bool inverse, const u64* src, size_t src_ls,
                  const std::vector<u32>* src_off) {
  if (slot_off.size() > (size_t)kMaxSlots) throw Error(AEGIS_EINVAL, "too many limbs in one NTT launch");
  NttLaunch L;
  std::memset(&L, 0, sizeof(L));
  L.base = base;
  L.lane_stride = lane_stride;
  L.nlanes = nlanes;
  L.nslots = (u32)slot_off.size();
  L.n = n;
  for (size_t i = 0; i < slot_off.size(); ++i) {
    L.slot_off[i] = slot_off[i];
    L.prime[i] = (unsigned char)primes[i];
  }
  L.tw = d_tw;
  L.scale = d_scale;
  if (src) {  // out-of-place inverse (v2): caller checked ntt_v2_active
    L.in_base = src;
    L.in_lane_stride = src_ls;
    for (size_t i = 0; i < slot_off.size(); ++i) L.in_slot_off[i] = src_off ? (*src_off)[i] : slot_off[i];
  }
  // grid.x holds rows * ctas_per_row; split very large batches
  const u32 max_rows = 1u << 20;
  for (u32 l0 = 0; l0 < nlanes; ) {
    u32 nl = std::max<u32>(1, std::min<u32>(nlanes - l0, max_rows / std::max<u32>(1, L.nslots)));
    NttLaunch Lb = L;
    Lb.base = base + (size_t)l0 * lane_stride;
    if (src) Lb.in_base = src + (size_t)l0 * src_ls;
    Lb.nlanes = nl;
    AEGIS_CHECK_CUDA(ntt_run(Lb, (int)log_n, inverse, stream));
    count(2);
    l0 += nl;
  }
}

void Context::basis_convert(const u64* src, size_t src_ls, const std::vector<u32>& src_off,
                            const std::vector<u32>& src_ext, u64* dst, size_t dst_ls,
                            const std::vector<u32>& dst_off, const std::vector<u32>& dst_ext, u32 lanes) {
  const Plan& pl = plan(src_ext, dst_ext);
  ConvIO io;
  std::memset(&io, 0, sizeof(io));
  io.src = src;
  io.src_lane_stride = src_ls;
  io.dst = dst;
  io.dst_lane_stride = dst_ls;
  for (size_t i = 0; i < src_off.size(); ++i) io.src_off[i] = src_off[i];
  for (size_t i = 0; i < dst_off.size(); ++i) io.dst_off[i] = dst_off[i];
  AEGIS_CHECK_CUDA(launch_basis_convert(pl.dev, pl.tables, io, lanes, n, pl.k, pl.m, stream));
  count();
}

// Exact conversion of `lanes` source sets followed by the forward NTT of the
// targets.  At N = 2^16 with <= 4 sources this is the fused path: one prep
// kernel (sources -> xt in place, overflow counts -> vbuf) and the NTT whose
// first pass computes the converted values itself (ntt.cu cfwd_a).  The
// sources are clobbered either way (callers pass scratch limbs).
bool Context::conv_ntt(u64* src, size_t src_ls, const std::vector<u32>& src_off, const std::vector<u32>& src_ext,
                       u64* dst, size_t dst_ls, const std::vector<u32>& dst_off, const std::vector<u32>& dst_ext,
                       u32 lanes, u64* vbuf, const NttFin* fin, bool lazy_out, bool pass_a_only) {
  const bool fused = log_n == 16 && g_ntt_impl == kNttF64 && g_ntt_v2 && g_conv_fused && src_off.size() <= 4 &&
                     dst_off.size() <= (size_t)kMaxSlots && vbuf != nullptr;
  if (!fused) {
    if (lazy_out || pass_a_only) throw Error(AEGIS_ELOGIC, "lazy / split NTT outputs need the fused conversion path");
    basis_convert(src, src_ls, src_off, src_ext, dst, dst_ls, dst_off, dst_ext, lanes);
    ntt(dst, dst_ls, lanes, dst_off, dst_ext, false);
    return false;
  }
  const Plan& pl = plan(src_ext, dst_ext);
  ConvIO io;
  std::memset(&io, 0, sizeof(io));
  io.src = src;
  io.src_lane_stride = src_ls;
  for (size_t i = 0; i < src_off.size(); ++i) io.src_off[i] = src_off[i];
  AEGIS_CHECK_CUDA(launch_conv_prep(pl.dev, pl.tables, io, vbuf, n, lanes, n, pl.k, pl.m, stream));
  count();
  NttLaunch L;
  std::memset(&L, 0, sizeof(L));
  L.base = dst;
  L.lane_stride = dst_ls;
  L.nlanes = lanes;
  L.nslots = (u32)dst_off.size();
  L.n = n;
  for (size_t i = 0; i < dst_off.size(); ++i) {
    L.slot_off[i] = dst_off[i];
    L.prime[i] = (unsigned char)dst_ext[i];
  }
  L.tw = d_tw;
  L.scale = d_scale;
  L.lazy_out = lazy_out ? 1u : 0u;
  NttConvIn c;
  std::memset(&c, 0, sizeof(c));
  c.plan = pl.dev;
  c.hat_tab = pl.tables;
  c.src = src;
  c.src_ls = src_ls;
  for (size_t i = 0; i < src_off.size(); ++i) c.src_off[i] = src_off[i];
  c.k = pl.k;
  c.v = vbuf;
  c.v_ls = n;
  AEGIS_CHECK_CUDA(ntt_conv_fwd(L, c, fin, stream, pass_a_only));
  count(pass_a_only ? 1 : 2);
  return fin != nullptr;
}

// ---------------------------------------------------------------------------
// Hybrid key switching, split so the ModUp can be hoisted:
//   modup()   Intt(d) -> per digit exact centred lift to Q_l u P -> Ntt
//             into ext[lane][digit][slot][n] (own-digit slots are not written:
//             the key product reads them straight from d)
//   ks_core() acc_c = sum_j ext_j * key[j][c]  ->  ModDown  ->  finish, where
//             finish optionally applies the eval-domain automorphism (Rot).
// ---------------------------------------------------------------------------
Context::KsShape Context::ks_shape(u32 l) const {
  KsShape s;
  s.l = l;
  s.ns = l + kAlpha;
  s.dn = (l + kAlpha - 1) / kAlpha;
  return s;
}

void Context::modup(const u64* d, size_t d_ls, u32 lanes, u32 l, u64* ext, bool pass_a_only) {
  if (l == 0 || l > chain) throw Error(AEGIS_EINVAL, "key switch level out of range");
  const KsShape S = ks_shape(l);
  const size_t ext_ls = modup_words_per_lane(l);
  std::vector<u32> main_off(l), main_ext(l);
  for (u32 i = 0; i < l; ++i) main_off[i] = main_ext[i] = i;
  const size_t budget = ws_budget(1);
  const u32 B = (u32)std::max<size_t>(1, std::min<size_t>(lanes, budget / ((size_t)l * n * 8)));
  u64* dc = alloc((size_t)B * (l + 1) * n);
  u64* vbuf = dc + (size_t)B * l * n;
  for (u32 l0 = 0; l0 < lanes; l0 += B) {
    const u32 nb = std::min(B, lanes - l0);
    if (ntt_v2_active((int)log_n)) {  // out-of-place INTT: d is read once, dc written once
      ntt(dc, (size_t)l * n, nb, main_off, main_ext, true, d + (size_t)l0 * d_ls, d_ls);
    } else {
      AEGIS_CHECK_CUDA(cudaMemcpy2DAsync(dc, (size_t)l * n * 8, d + (size_t)l0 * d_ls, d_ls * 8, (size_t)l * n * 8, nb,
                                         cudaMemcpyDeviceToDevice, stream));
      ntt(dc, (size_t)l * n, nb, main_off, main_ext, true);
    }
    for (u32 j = 0; j < S.dn; ++j) {
      const u32 lo = j * kAlpha, hi = std::min(l, lo + kAlpha);
      std::vector<u32> s_off, s_ext, t_off, t_ext;
      for (u32 i = lo; i < hi; ++i) { s_off.push_back(i); s_ext.push_back(i); }
      // compact layout: digit j stores only its ns - |D_j| target slots
      for (u32 t = 0; t < S.ns; ++t)
        if (t < lo || t >= hi) {
          t_off.push_back((u32)t_off.size());
          t_ext.push_back(t < l ? t : kSpecialBase + (t - l));
        }
      u64* ej = ext + (size_t)l0 * ext_ls + (size_t)(j * S.ns - lo) * n;
      conv_ntt(dc, (size_t)l * n, s_off, s_ext, ej, ext_ls, t_off, t_ext, nb, vbuf, nullptr, modup_lazy(), pass_a_only);
    }
  }
  release(dc);
}

void Context::ks_core(const u64* ext, const u64* d, size_t d_ls, u32 lanes, u32 l, const u64* kbase, u64 galois,
                      const KsOut& o, bool ext_pass_a) {
  const KsShape S = ks_shape(l);
  const u32 K = kAlpha, ns = S.ns;
  const size_t ext_ls = modup_words_per_lane(l), acc_ls = (size_t)2 * ns * n;
  std::vector<u32> main_off(l), main_ext(l);
  for (u32 i = 0; i < l; ++i) main_off[i] = main_ext[i] = i;
  const size_t per_lane = (size_t)n * (2 * ns + 2 * (size_t)l);
  const size_t budget = ws_budget(1);
  const u32 B = (u32)std::max<size_t>(1, std::min<size_t>(lanes, budget / (per_lane * 8)));
  u64* acc = alloc((per_lane + 2 * (size_t)n) * B);  // [B][2][ns][n]
  u64* pcv = acc + (size_t)B * 2 * ns * n;        // [B][2][l][n]
  u64* vbuf = pcv + (size_t)B * 2 * l * n;        // [2B][n]
  // constants of the finish step: P^{-1} mod q_i
  FinishIO f;
  std::memset(&f, 0, sizeof(f));
  f.comps = 1;
  f.limbs = l;
  f.galois = galois;
  f.log_n = log_n;
  for (u32 i = 0; i < l; ++i) {
    const u64 q = prime(i);
    u64 P = 1;
    for (u32 k = 0; k < K; ++k) P = h_mulmod(P, prime(kSpecialBase + k) % q, q);
    f.ext[i] = i;
    f.f[i] = h_inv(P, q);
    f.f_p[i] = h_shoup(f.f[i], q);
  }
  KeyMulIO km;
  std::memset(&km, 0, sizeof(km));
  km.key = kbase;
  km.key_slots = key_slots();
  km.level = l;
  km.dnum = S.dn;
  km.nslots = ns;
  for (u32 t = 0; t < ns; ++t) {
    km.slot_ext[t] = t < l ? t : kSpecialBase + (t - l);
    km.slot_key[t] = t < l ? t : chain + (t - l);
  }
  std::vector<u32> p_off, p_ext, ps_off(K), ps_ext(K);
  for (u32 c = 0; c < 2; ++c)
    for (u32 k = 0; k < K; ++k) { p_off.push_back(c * ns + l + k); p_ext.push_back(kSpecialBase + k); }
  for (u32 k = 0; k < K; ++k) { ps_off[k] = l + k; ps_ext[k] = kSpecialBase + k; }

  for (u32 l0 = 0; l0 < lanes; l0 += B) {
    const u32 nb = std::min(B, lanes - l0);
    // KeyMul inner product over digits
    km.ext = ext + (size_t)l0 * ext_ls;
    km.ext_lane_stride = ext_ls;
    km.d = d + (size_t)l0 * d_ls;
    km.d_lane_stride = d_ls;
    km.acc = acc;
    km.acc_lane_stride = acc_ls;
    km.ext_lazy = modup_lazy() ? 1u : 0u;
    if (ext_pass_a) {  // ModUp second pass fused with the key product (ntt.cu fwd_b_km)
      KmB kb;
      std::memset(&kb, 0, sizeof(kb));
      kb.ext = km.ext;
      kb.ext_ls = ext_ls;
      kb.d = km.d;
      kb.d_ls = d_ls;
      kb.key = kbase;
      kb.acc = acc;
      kb.acc_ls = acc_ls;
      kb.tw = d_tw;
      kb.scale = d_scale;
      kb.key_slots = key_slots();
      kb.level = l;
      kb.dnum = S.dn;
      kb.nslots = ns;
      kb.chain = chain;
      kb.nlanes = nb;
      kb.n = n;
      AEGIS_CHECK_CUDA(ntt_fwd_b_keymul(kb, stream));
    } else {
      AEGIS_CHECK_CUDA(launch_keymul(km, nb, n, d_pc, stream));
    }
    count();
    // ModDown: Intt the P limbs, exact lift P -> Q_l, Ntt, (acc - conv) * P^{-1}
    ntt(acc, acc_ls, nb, p_off, p_ext, true);
    // (lane, comp) pairs are uniform "virtual lanes" of stride ns*n / l*n;
    // the finish (acc_Q - conv) * P^{-1} + add (+ automorphism) is fused into
    // the last NTT pass when available
    NttFin fin;
    std::memset(&fin, 0, sizeof(fin));
    fin.x = acc;
    fin.x_lane = (long long)acc_ls;
    fin.x_comp = (long long)ns * n;
    fin.add = o.add[0] ? o.add[0] + (size_t)l0 * o.add_lane[0] : nullptr;
    fin.add_lane = (long long)o.add_lane[0];
    fin.add_comp = o.add[1] ? (long long)(o.add[1] - o.add[0]) : 0;
    fin.add_comps = o.add[1] ? 2 : 1;
    fin.out = o.out[0] + (size_t)l0 * o.out_lane[0];
    fin.out_lane = (long long)o.out_lane[0];
    fin.out_comp = (long long)(o.out[1] - o.out[0]);
    fin.comps = 2;
    fin.galois = galois;
    fin.galois_inv = galois <= 1 ? 1 : h_powmod(galois, (u64)n - 1, 2ull * n);
    fin.log_n = log_n;
    for (u32 i = 0; i < l; ++i) fin.f[i] = f.f[i];
    const bool uniform = o.out_lane[0] == o.out_lane[1] && (!o.add[1] || o.add_lane[0] == o.add_lane[1]);
    if (conv_ntt(acc, (size_t)ns * n, ps_off, ps_ext, pcv, (size_t)l * n, main_off, main_ext, 2 * nb, vbuf,
                 uniform ? &fin : nullptr))
      continue;  // finished inside the NTT
    for (u32 c = 0; c < 2; ++c) {
      f.x = acc + (size_t)c * ns * n;
      f.x_lane = acc_ls;
      f.y = pcv + (size_t)c * l * n;
      f.y_lane = (size_t)2 * l * n;
      f.add = o.add[c] ? o.add[c] + (size_t)l0 * o.add_lane[c] : nullptr;
      f.add_lane = o.add_lane[c];
      f.out = o.out[c] + (size_t)l0 * o.out_lane[c];
      f.out_lane = o.out_lane[c];
      AEGIS_CHECK_CUDA(launch_finish(f, nb, n, d_pc, stream));
      count();
    }
  }
  release(acc);
}

void Context::keyswitch(const u64* d, size_t d_ls, u32 lanes, u32 l, u64 key_id, const KsOut& o, u64 galois) {
  const size_t ext_lane = modup_words_per_lane(l);
  const u32 B = (u32)std::max<size_t>(1, std::min<size_t>(lanes, ws_budget(2) / (ext_lane * 8)));
  u64* ext = alloc(ext_lane * B);
  const u64* kbase = key(key_id);
  // not hoisted: ModUp's second NTT pass runs inside the key product (the
  // ModUp limbs are never materialised)
  const bool split = modup_lazy() && g_km_split;
  for (u32 l0 = 0; l0 < lanes; l0 += B) {
    const u32 nb = std::min(B, lanes - l0);
    modup(d + (size_t)l0 * d_ls, d_ls, nb, l, ext, split);
    KsOut ob = o;
    for (int c = 0; c < 2; ++c) {
      ob.out[c] = o.out[c] + (size_t)l0 * o.out_lane[c];
      if (o.add[c]) ob.add[c] = o.add[c] + (size_t)l0 * o.add_lane[c];
    }
    ks_core(ext, d + (size_t)l0 * d_ls, d_ls, nb, l, kbase, galois, ob, split);
  }
  release(ext);
}

// ---------------------------------------------------------------------------
// HE operators
// ---------------------------------------------------------------------------
void Context::op_rot(Bundle& out, u32 out_lane, const Bundle& in, LaneMap im, u32 lanes, u32 level, int offset) {
  op_rot_cached(out, out_lane, in, im, lanes, level, offset, nullptr);
}

// Rot_r(c0, c1) = (auto(c0) + KS_0(auto(c1)), KS_1(auto(c1)))
//              = auto(c0 + MD_0, MD_1),  MD = ModDown(sum_j ModUp(c1)_j key'_r,j)
// (rotation keys are stored pre-permuted, see generate_key).  `ext` may hold
// ModUp(c1) of these lanes already (hoisting across the rotations of one
// source); otherwise it is computed here.
void Context::op_rot_cached(Bundle& out, u32 out_lane, const Bundle& in, LaneMap im, u32 lanes, u32 level,
                            int offset, const u64* ext) {
  if (level > in.level || level > out.level) throw Error(AEGIS_EINVAL, "rotation level exceeds operand level");
  const u64 gk = galois_of(offset);
  const u64 key_id = rotation_key_id(offset);
  const size_t in_ls = (size_t)in.comps * in.level * n;
  KsOut o;
  o.out_lane[0] = o.out_lane[1] = (size_t)out.comps * out.level * n;
  o.add_lane[0] = o.add_lane[1] = in_ls;
  o.add[1] = nullptr;
  if (im.count != lanes) {  // wrapped operand lanes: one lane at a time
    if (ext) throw Error(AEGIS_ELOGIC, "hoisted rotation needs aligned lanes");
    for (u32 l = 0; l < lanes; ++l) {
      const u32 il = im.at(l, lanes);
      o.out[0] = out.view().limb(out_lane + l, 0, 0, n);
      o.out[1] = out.view().limb(out_lane + l, 1, 0, n);
      o.add[0] = in.view().limb(il, 0, 0, n);
      keyswitch(in.view().limb(il, 1, 0, n), in_ls, 1, level, key_id, o, gk);
    }
    return;
  }
  o.out[0] = out.view().limb(out_lane, 0, 0, n);
  o.out[1] = out.view().limb(out_lane, 1, 0, n);
  o.add[0] = in.view().limb(im.lane0, 0, 0, n);
  const u64* c1 = in.view().limb(im.lane0, 1, 0, n);
  if (ext) {
    ks_core(ext, c1, in_ls, lanes, level, key(key_id), gk, o);
  } else {
    keyswitch(c1, in_ls, lanes, level, key_id, o, gk);
  }
}

void Context::op_relin(Bundle& b, u32 lane, u32 lanes, u32 level) {
  if (b.comps < 3) throw Error(AEGIS_ELOGIC, "relinearisation needs a 3-component product");
  const size_t ls = (size_t)b.comps * b.level * n;
  KsOut o;
  o.out[0] = b.view().limb(lane, 0, 0, n);
  o.out[1] = b.view().limb(lane, 1, 0, n);
  o.add[0] = o.out[0];
  o.add[1] = o.out[1];
  o.out_lane[0] = o.out_lane[1] = o.add_lane[0] = o.add_lane[1] = ls;
  keyswitch(b.view().limb(lane, 2, 0, n), ls, lanes, level, 0, o);
}

void Context::op_rescale(Bundle& out, u32 out_lane, const Bundle& in, LaneMap im, u32 lanes, u32 L) {
  if (L < 2) throw Error(AEGIS_EINVAL, "level underflow: cannot rescale below level 1");
  if (im.count != lanes) throw Error(AEGIS_ELOGIC, "rescale operand lanes must match");
  const u32 m = L - 1;
  // lanes in batches so the workspace stays ~1 GB (a T=2048 score tensor is 50 GB)
  const size_t per_lane = (size_t)2 * n * (1 + m);
  const u32 B = (u32)std::max<size_t>(1, std::min<size_t>(lanes, ws_budget(1) / (per_lane * 8)));
  u64* last = alloc((size_t)2 * B * n);
  u64* conv = alloc((size_t)2 * B * (m + 1) * n);
  u64* vbuf = conv + (size_t)2 * B * m * n;
  std::vector<u32> off(m), ext(m);
  for (u32 i = 0; i < m; ++i) off[i] = ext[i] = i;
  FinishIO f;
  std::memset(&f, 0, sizeof(f));
  f.x_lane = (size_t)in.comps * in.level * n;
  f.x_comp = (size_t)in.level * n;
  f.y = conv;
  f.y_lane = (size_t)2 * m * n;
  f.y_comp = (size_t)m * n;
  f.out_lane = (size_t)out.comps * out.level * n;
  f.out_comp = (size_t)out.level * n;
  f.comps = 2;
  f.limbs = m;
  const u64 ql = prime(L - 1);
  for (u32 i = 0; i < m; ++i) {
    const u64 q = prime(i);
    f.ext[i] = i;
    f.f[i] = h_inv(ql % q, q);
    f.f_p[i] = h_shoup(f.f[i], q);
  }
  for (u32 l0 = 0; l0 < lanes; l0 += B) {
    const u32 nb = std::min(B, lanes - l0);
    // last limb of every (lane, comp) -> [lane][comp][n], Intt, centred lift to q_0..q_{L-2}, Ntt
    const bool v2 = ntt_v2_active((int)log_n) && in.comps == 2;
    if (v2) {  // (lane, comp) are uniform virtual lanes of stride level*n when comps == 2
      const std::vector<u32> src_off{L - 1};
      ntt(last, n, 2 * nb, {0}, {L - 1}, true, in.view().limb(im.lane0 + l0, 0, 0, n), (size_t)in.level * n, &src_off);
    } else {
      AEGIS_CHECK_CUDA(launch_copy(View{last, nb, 2, 1}, 0, in.view(), LaneMap{im.lane0 + l0, nb}, nb, 2, 1, L - 1, n,
                                   stream));
      count();
      ntt(last, n, 2 * nb, {0}, {L - 1}, true);
    }
    // out_i = (x_i - r_i) * q_{L-1}^{-1}   (div_round on the centred value, rns_math.hpp:196-202),
    // fused into the conversion NTT's last pass when available
    f.x = in.view().limb(im.lane0 + l0, 0, 0, n);
    f.out = out.view().limb(out_lane + l0, 0, 0, n);
    NttFin fin;
    std::memset(&fin, 0, sizeof(fin));
    fin.x = f.x;
    fin.x_lane = (long long)f.x_lane;
    fin.x_comp = (long long)f.x_comp;
    fin.out = f.out;
    fin.out_lane = (long long)f.out_lane;
    fin.out_comp = (long long)f.out_comp;
    fin.comps = 2;
    fin.galois_inv = 1;
    fin.log_n = log_n;
    for (u32 i = 0; i < m; ++i) fin.f[i] = f.f[i];
    if (conv_ntt(last, n, {0}, {L - 1}, conv, (size_t)m * n, off, ext, 2 * nb, vbuf, &fin)) continue;
    AEGIS_CHECK_CUDA(launch_finish(f, nb, n, d_pc, stream));
    count();
  }
  release(last);
  release(conv);
}

void Context::op_boot(Bundle& out, u32 out_lane, const Bundle& in, LaneMap im, u32 lanes, u32 L, u32 out_level) {
  if (im.count != lanes) throw Error(AEGIS_ELOGIC, "boot operand lanes must match");
  const u32 keep = std::min(L, out_level);
  AEGIS_CHECK_CUDA(launch_copy(out.view(), out_lane, in.view(), im, lanes, 2, keep, 0, n, stream));
  count();
  if (out_level <= L) return;
  // value-preserving lift: Intt(Q_L) -> exact centred lift -> new limbs -> Ntt
  u64* xc = alloc((size_t)2 * lanes * L * n);
  AEGIS_CHECK_CUDA(launch_copy(View{xc, lanes, 2, L}, 0, in.view(), im, lanes, 2, L, 0, n, stream));
  count();
  std::vector<u32> soff(L), sext(L);
  for (u32 i = 0; i < L; ++i) soff[i] = sext[i] = i;
  ntt(xc, (size_t)L * n, 2 * lanes, soff, sext, true);
  std::vector<u32> toff, text;
  for (u32 i = L; i < out_level; ++i) { toff.push_back(i); text.push_back(i); }
  // virtual lanes (lane, comp): out stride is uniform only when comps == 2
  if (out.comps == 2) {
    basis_convert(xc, (size_t)L * n, soff, sext, out.view().limb(out_lane, 0, 0, n), (size_t)out.level * n, toff,
                  text, 2 * lanes);
    ntt(out.view().limb(out_lane, 0, 0, n), (size_t)out.level * n, 2 * lanes, toff, text, false);
  } else {
    for (u32 c = 0; c < 2; ++c) {
      basis_convert(xc + (size_t)c * L * n, (size_t)2 * L * n, soff, sext, out.view().limb(out_lane, c, 0, n),
                    (size_t)out.comps * out.level * n, toff, text, lanes);
      ntt(out.view().limb(out_lane, c, 0, n), (size_t)out.comps * out.level * n, lanes, toff, text, false);
    }
  }
  release(xc);
}

void Context::op_cmult(Bundle& out, u32 out_lane, u32 lanes, const Bundle& a, LaneMap ma, const Bundle& b,
                       LaneMap mb, u32 level) {
  if (out.comps < 3) throw Error(AEGIS_ELOGIC, "CMult output needs 3 components");
  AEGIS_CHECK_CUDA(launch_cmult(out.view(), out_lane, a.view(), ma, b.view(), mb, lanes, level, n, d_pc, stream));
  count();
}

void Context::op_cadd(Bundle& out, u32 out_lane, u32 lanes, const Bundle& a, LaneMap ma, const Bundle* b,
                      LaneMap mb, u32 level, bool acc) {
  if (!acc && !b) throw Error(AEGIS_ELOGIC, "CAdd needs two operands");
  AEGIS_CHECK_CUDA(launch_cadd(out.view(), out_lane, a.view(), ma, b ? b->view() : a.view(), mb, acc, lanes, 2,
                               level, n, d_pc, stream));
  count();
}

void Context::op_pmult(Bundle& acc, u32 acc_lane, u32 acc_lanes, u32 chunk_period, const Bundle& x, u32 x_lane,
                       u32 x_lanes, u32 wbundle, u32 wlanes, u32 level, u32 t_lo, u32 t_hi, u32 ci_lo,
                       u32 ci_hi, const Bundle* wst, u32 w_lane0, u32 o_lo, u32 o_cnt) {
  const PcmmShape sh = pcmm_shape(x_lanes, acc_lanes, wlanes, chunk_period);
  t_hi = std::min(t_hi, sh.tg);
  ci_hi = std::min(ci_hi, sh.c_in);
  if (t_lo >= t_hi || ci_lo >= ci_hi) return;
  if (wst && (wst->comps != 1 || wst->level < level || (uint64_t)w_lane0 + wlanes > wst->lanes))
    throw Error(AEGIS_EINVAL, "stored PMult weights: need a 1-component bundle covering the weight lanes and level");
  u64* rk = nullptr;
  if (!wst) {
    rk = alloc((size_t)wlanes * level);
    AEGIS_CHECK_CUDA(launch_weight_rowkeys(rk, wlanes, level, seed_weight, wbundle, stream));
    count();
  }
  for (u32 s = 0; s < sh.S; ++s) {
    // sub-tensor s occupies acc lanes [s*chunk, (s+1)*chunk), token-major inside
    PmultArgs a;
    a.acc = acc.view();
    const u32 olo = std::min(o_lo, sh.c_sub), ocnt = std::min(o_cnt, sh.c_sub - olo);
    if (!ocnt) continue;
    a.acc_lane0 = acc_lane + pcmm_lane(sh, t_lo, s * sh.c_sub + olo);
    a.acc_tstride = sh.S == 1 ? sh.c_out : sh.c_sub;
    a.x = x.view();
    a.x_lane0 = x_lane + t_lo * sh.c_in + ci_lo;
    a.x_tstride = sh.c_in;
    a.tg = t_hi - t_lo;
    a.c_in = ci_hi - ci_lo;
    a.c_out = ocnt;
    a.ci_off = ci_lo;
    a.o_off = s * sh.c_sub + olo;
    a.w_cout = sh.c_out;
    a.limbs = level;
    a.n = n;
    a.rowkeys = rk;
    if (wst) {
      a.wst = wst->view();
      a.w_lane0 = w_lane0;
    }
    AEGIS_CHECK_CUDA(launch_pmult_acc(a, d_pc, stream));
    count((a.tg + 3) / 4);
  }
  release(rk);
}

}  // namespace aegis

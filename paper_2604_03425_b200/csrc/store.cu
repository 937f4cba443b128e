// store.cu -- wire / disk format of encoded plaintexts, ciphertext bundles and
// key-switching keys, with streaming transfer (the
// paper's pre-encoded weights, ~700 GB at 2048 tokens
// PAPER.md:84, and the keys of ckks.hpp:217-223 do not fit in HBM together,
// so they arrive from host storage while the GPU computes).
//
// File = 128-byte header + payload of little-endian u64 residues:
//   magic "AEGS", version 1, kind (0 = bundle, 1 = key), log_n, chain,
//   lanes|digits, comps, levels|slots, prime-chain fingerprint, key id,
//   payload words, content hash (DESIGN.md §2.4 over the payload as a
//   [lanes][comps][levels][N] array), flags (bit 0: rotation key stored
//   pre-permuted, the library's internal form).
// Bundles are [lane][comp][limb][N] canonical residues (include/aegis.h);
// keys are [digit][comp][slot][N] in the internal layout (NTT domain,
// rotation keys pre-permuted), i.e. exactly what aegis_keys_generate /
// aegis_keys_upload leave on the device.
//
// Streaming: the payload moves in 64 MiB chunks through two pinned staging
// buffers; while one chunk's DMA runs on the compute stream the host reads
// (or writes) the other, so disk / page-cache bandwidth and PCIe overlap.
// After a load the content hash is recomputed on the device and compared
// with the header (a torn or foreign file is rejected, nothing is kept).
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

#include "context.h"
#include "store.h"

namespace aegis {

namespace {

constexpr char kMagic[4] = {'A', 'E', 'G', 'S'};
constexpr size_t kChunk = (size_t)64 << 20;

struct Header {
  char magic[4];
  u32 version, kind, log_n, chain, lanes, comps, levels;
  u64 fingerprint, key_id, words, hash, flags;
  unsigned char pad[128 - 4 - 7 * 4 - 5 * 8];
};
static_assert(sizeof(Header) == 128, "header size");

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};

struct Pinned {
  void* p[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  Pinned() {
    for (int i = 0; i < 2; ++i) {
      AEGIS_CHECK_CUDA(cudaMallocHost(&p[i], kChunk));
      AEGIS_CHECK_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
  }
  ~Pinned() {
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) cudaEventDestroy(ev[i]);
      if (p[i]) cudaFreeHost(p[i]);
    }
  }
};

u64 device_hash(Context& c, const u64* dev, u32 lanes, u32 comps, u32 levels) {
  unsigned long long* d = nullptr;
  AEGIS_CHECK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), 8, c.stream));
  AEGIS_CHECK_CUDA(cudaMemsetAsync(d, 0, 8, c.stream));
  AEGIS_CHECK_CUDA(launch_hash(View{const_cast<u64*>(dev), lanes, comps, levels}, 0, lanes, comps, levels, c.n, d,
                               c.stream));
  c.count();
  unsigned long long h = 0;
  AEGIS_CHECK_CUDA(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, c.stream));
  AEGIS_CHECK_CUDA(cudaFreeAsync(d, c.stream));
  AEGIS_CHECK_CUDA(cudaStreamSynchronize(c.stream));
  return h;
}

void write_payload(Context& c, FILE* f, const u64* dev, size_t words, const std::string& path) {
  Pinned pin;
  const size_t per = kChunk / 8;
  size_t nchunks = (words + per - 1) / per;
  // D2H of chunk k+1 overlaps the fwrite of chunk k
  auto issue = [&](size_t k) {
    const size_t off = k * per, cnt = std::min(per, words - off);
    AEGIS_CHECK_CUDA(cudaMemcpyAsync(pin.p[k & 1], dev + off, cnt * 8, cudaMemcpyDeviceToHost, c.stream));
    AEGIS_CHECK_CUDA(cudaEventRecord(pin.ev[k & 1], c.stream));
  };
  if (nchunks) issue(0);
  for (size_t k = 0; k < nchunks; ++k) {
    if (k + 1 < nchunks) issue(k + 1);
    AEGIS_CHECK_CUDA(cudaEventSynchronize(pin.ev[k & 1]));
    const size_t cnt = std::min(per, words - k * per);
    if (std::fwrite(pin.p[k & 1], 8, cnt, f) != cnt) throw Error(AEGIS_EINVAL, "short write to " + path);
  }
}

void read_payload(Context& c, FILE* f, u64* dev, size_t words, const std::string& path) {
  Pinned pin;
  const size_t per = kChunk / 8;
  const size_t nchunks = (words + per - 1) / per;
  for (size_t k = 0; k < nchunks; ++k) {
    const int b = (int)(k & 1);
    if (k >= 2) AEGIS_CHECK_CUDA(cudaEventSynchronize(pin.ev[b]));  // its previous DMA has drained
    const size_t off = k * per, cnt = std::min(per, words - off);
    if (std::fread(pin.p[b], 8, cnt, f) != cnt) throw Error(AEGIS_EINVAL, "truncated payload in " + path);
    AEGIS_CHECK_CUDA(cudaMemcpyAsync(dev + off, pin.p[b], cnt * 8, cudaMemcpyHostToDevice, c.stream));
    AEGIS_CHECK_CUDA(cudaEventRecord(pin.ev[b], c.stream));
  }
  AEGIS_CHECK_CUDA(cudaStreamSynchronize(c.stream));
}

Header read_header(Context& c, FILE* f, const std::string& path, u32 kind) {
  Header h;
  if (std::fread(&h, sizeof(h), 1, f) != 1) throw Error(AEGIS_EINVAL, "cannot read header of " + path);
  if (std::memcmp(h.magic, kMagic, 4) || h.version != 1) throw Error(AEGIS_EINVAL, path + " is not an aegis store file");
  if (h.kind != kind) throw Error(AEGIS_EINVAL, path + (kind ? " holds a bundle, not a key" : " holds a key, not a bundle"));
  if (h.log_n != c.log_n || h.chain != c.chain || h.fingerprint != c.chain_fingerprint())
    throw Error(AEGIS_EINVAL, path + " was written under a different ring / prime chain");
  if (h.words != (u64)h.lanes * h.comps * h.levels * c.n) throw Error(AEGIS_EINVAL, path + ": inconsistent header");
  return h;
}

}  // namespace

void store_save_bundle(Context& c, const Bundle& b, const std::string& path) {
  File f;
  f.f = std::fopen(path.c_str(), "wb");
  if (!f.f) throw Error(AEGIS_EINVAL, "cannot open " + path + " for writing");
  Header h{};
  std::memcpy(h.magic, kMagic, 4);
  h.version = 1;
  h.kind = 0;
  h.log_n = c.log_n;
  h.chain = c.chain;
  h.lanes = b.lanes;
  h.comps = b.comps;
  h.levels = b.level;
  h.fingerprint = c.chain_fingerprint();
  h.words = (u64)b.lanes * b.comps * b.level * c.n;
  h.hash = device_hash(c, b.ptr, b.lanes, b.comps, b.level);
  if (std::fwrite(&h, sizeof(h), 1, f.f) != 1) throw Error(AEGIS_EINVAL, "short write to " + path);
  write_payload(c, f.f, b.ptr, h.words, path);
  if (std::fflush(f.f)) throw Error(AEGIS_EINVAL, "cannot flush " + path);
}

Bundle* store_load_bundle(Context& c, const std::string& path) {
  File f;
  f.f = std::fopen(path.c_str(), "rb");
  if (!f.f) throw Error(AEGIS_EINVAL, "cannot open " + path);
  const Header h = read_header(c, f.f, path, 0);
  if (!h.lanes || !h.comps || h.comps > 3 || !h.levels || h.levels > c.chain)
    throw Error(AEGIS_EINVAL, path + ": bad bundle shape");
  Bundle* b = c.new_bundle(h.lanes, h.comps, h.levels, false);
  try {
    read_payload(c, f.f, b->ptr, h.words, path);
    if (device_hash(c, b->ptr, b->lanes, b->comps, b->level) != h.hash)
      throw Error(AEGIS_EINVAL, path + ": content hash mismatch (torn or corrupted file)");
  } catch (...) {
    c.free_bundle(b);
    throw;
  }
  return b;
}

void store_save_key(Context& c, u64 key_id, const std::string& path) {
  const u64* k = c.key_storage(key_id, false);
  if (!k) throw Error(AEGIS_EINVAL, "no key " + std::to_string(key_id) + " on this context");
  File f;
  f.f = std::fopen(path.c_str(), "wb");
  if (!f.f) throw Error(AEGIS_EINVAL, "cannot open " + path + " for writing");
  Header h{};
  std::memcpy(h.magic, kMagic, 4);
  h.version = 1;
  h.kind = 1;
  h.log_n = c.log_n;
  h.chain = c.chain;
  h.lanes = c.key_digits();
  h.comps = 2;
  h.levels = c.key_slots();
  h.fingerprint = c.chain_fingerprint();
  h.key_id = key_id;
  h.words = c.key_bytes() / 8;
  h.hash = device_hash(c, k, h.lanes, 2, h.levels);
  h.flags = key_id >= 500 ? 1 : 0;  // rotation keys: internal pre-permuted form
  if (std::fwrite(&h, sizeof(h), 1, f.f) != 1) throw Error(AEGIS_EINVAL, "short write to " + path);
  write_payload(c, f.f, k, h.words, path);
  if (std::fflush(f.f)) throw Error(AEGIS_EINVAL, "cannot flush " + path);
}

void store_load_key(Context& c, u64 key_id, const std::string& path) {
  File f;
  f.f = std::fopen(path.c_str(), "rb");
  if (!f.f) throw Error(AEGIS_EINVAL, "cannot open " + path);
  const Header h = read_header(c, f.f, path, 1);
  if (h.lanes != c.key_digits() || h.comps != 2 || h.levels != c.key_slots())
    throw Error(AEGIS_EINVAL, path + ": key shape does not match this context");
  if ((h.key_id >= 500) != (key_id >= 500))
    throw Error(AEGIS_EINVAL, path + ": rotation and relinearisation keys are stored in different forms");
  c.drop_key(key_id);  // a failed load leaves no key behind (the next use regenerates or errors)
  u64* k = c.key_storage(key_id, true);
  try {
    read_payload(c, f.f, k, h.words, path);
    if (device_hash(c, k, h.lanes, 2, h.levels) != h.hash)
      throw Error(AEGIS_EINVAL, path + ": content hash mismatch (torn or corrupted file)");
  } catch (...) {
    c.drop_key(key_id);
    throw;
  }
}

}  // namespace aegis

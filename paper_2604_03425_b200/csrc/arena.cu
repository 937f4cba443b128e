// arena.cu -- see arena.h.
#include "arena.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>

namespace aegis {

namespace {
// driver entry points resolved through the runtime (no link-time libcuda
// dependency: the library must load on hosts without a driver)
struct Drv {
  CUresult (*granularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*addr_free)(CUdeviceptr, size_t) = nullptr;
  CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*release)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  bool ok = false;
};
template <class F>
bool entry(const char* name, F& f) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess || !p)
    return false;
  f = reinterpret_cast<F>(p);
  return true;
}
const Drv& drv() {
  static Drv d = [] {
    Drv r;
    r.ok = entry("cuMemGetAllocationGranularity", r.granularity) && entry("cuMemAddressReserve", r.reserve) &&
           entry("cuMemAddressFree", r.addr_free) && entry("cuMemCreate", r.create) &&
           entry("cuMemRelease", r.release) && entry("cuMemMap", r.map) && entry("cuMemUnmap", r.unmap) &&
           entry("cuMemSetAccess", r.access);
    return r;
  }();
  return d;
}
constexpr size_t kAlign = (size_t)64 << 10;     // allocation granularity inside the arena
constexpr size_t kMinChunk = (size_t)1 << 30;   // physical memory is mapped >= 1 GiB at a time
size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
}  // namespace

Arena::Arena(int device) : dev_(device) {
  if (!drv().ok) return;  // no VMM: alloc() returns nullptr and callers report OOM
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  if (drv().granularity(&gran_, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS) gran_ = 2 << 20;
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  reserve_ = round_up(tot + ((size_t)8 << 30), gran_);
  if (drv().reserve(&base_, reserve_, 0, 0, 0) != CUDA_SUCCESS) {
    base_ = 0;
    reserve_ = 0;
  }
}

Arena::~Arena() {
  if (!base_) return;
  for (auto it = chunks_.rbegin(); it != chunks_.rend(); ++it) {
    drv().unmap(base_ + it->off, it->size);
    drv().release(it->h);
  }
  drv().addr_free(base_, reserve_);
}

bool Arena::grow(size_t need) {
  if (!base_) return false;
  size_t sz = round_up(std::max(need, kMinChunk), gran_);
  for (int attempt = 0; attempt < 2; ++attempt) {
    if (mapped_ + sz > reserve_) sz = round_up(need, gran_);
    if (mapped_ + sz > reserve_) return false;
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = dev_;
    CUmemGenericAllocationHandle h;
    if (drv().create(&h, sz, &prop, 0) != CUDA_SUCCESS) {
      sz = round_up(need, gran_);  // retry with exactly what is needed
      continue;
    }
    if (drv().map(base_ + mapped_, sz, 0, h, 0) != CUDA_SUCCESS) {
      drv().release(h);
      return false;
    }
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = dev_;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    if (drv().access(base_ + mapped_, sz, &acc, 1) != CUDA_SUCCESS) {
      drv().unmap(base_ + mapped_, sz);
      drv().release(h);
      return false;
    }
    chunks_.push_back(Chunk{mapped_, sz, h});
    if (std::getenv("AEGIS_DEBUG"))
      fprintf(stderr, "[aegis] arena grow +%zu MiB -> %zu MiB mapped (request %zu MiB)\n", sz >> 20, (mapped_ + sz) >> 20,
              need >> 20);
    // new space joins the free block at the tail, if any
    size_t off = mapped_, len = sz;
    if (!free_.empty()) {
      auto last = std::prev(free_.end());
      if (last->first + last->second == mapped_) {
        off = last->first;
        len += last->second;
        free_.erase(last);
      }
    }
    free_[off] = len;
    mapped_ += sz;
    return true;
  }
  return false;
}

void* Arena::alloc(size_t bytes) {
  if (!base_) return nullptr;
  const size_t sz = round_up(std::max<size_t>(bytes, 1), kAlign);
  auto best = free_.end();
  for (auto it = free_.begin(); it != free_.end(); ++it)
    if (it->second >= sz && (best == free_.end() || it->second < best->second)) best = it;
  if (best == free_.end()) {
    size_t tail = 0;
    if (!free_.empty()) {
      auto last = std::prev(free_.end());
      if (last->first + last->second == mapped_) tail = last->second;
    }
    if (!grow(sz - tail)) return nullptr;
    best = std::prev(free_.end());
    if (best->second < sz) return nullptr;
  }
  const size_t off = best->first, len = best->second;
  free_.erase(best);
  if (len > sz) free_[off + sz] = len - sz;
  used_[off] = sz;
  in_use_ += sz;
  return (void*)(base_ + off);
}

void Arena::free(void* p) {
  const size_t off = (size_t)((CUdeviceptr)p - base_);
  auto u = used_.find(off);
  if (u == used_.end()) return;
  size_t o = off, len = u->second;
  in_use_ -= len;
  used_.erase(u);
  auto next = free_.lower_bound(o);
  if (next != free_.end() && o + len == next->first) {
    len += next->second;
    next = free_.erase(next);
  }
  if (next != free_.begin()) {
    auto prev = std::prev(next);
    if (prev->first + prev->second == o) {
      o = prev->first;
      len += prev->second;
      free_.erase(prev);
    }
  }
  free_[o] = len;
}

size_t Arena::largest_free() const {
  size_t m = 0;
  for (auto& kv : free_) m = std::max(m, kv.second);
  return m;
}

void Arena::trim() {
  if (free_.empty()) return;
  auto last = std::prev(free_.end());
  if (last->first + last->second != mapped_) return;
  size_t tail_start = last->first;
  while (!chunks_.empty() && chunks_.back().off >= tail_start) {
    const Chunk c = chunks_.back();
    chunks_.pop_back();
    drv().unmap(base_ + c.off, c.size);
    drv().release(c.h);
    mapped_ = c.off;
  }
  free_.erase(last);
  if (tail_start < mapped_) free_[tail_start] = mapped_ - tail_start;
}

}  // namespace aegis

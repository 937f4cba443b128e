// arena.h -- device memory arena for ciphertext bundles and key-switch workspaces.
//
// A layer at T = 2048 allocates and frees bundles of up to ~60 GB in a
// pattern the CUDA stream-ordered pool serves badly: a request that no cached
// block fits makes the pool map fresh physical memory, and near the 180 GB
// limit that means trimming and re-mapping tens of GB (hundreds of ms per op).
// The arena reserves one virtual range per context and maps physical memory
// into it in large chunks as the high-water mark grows (cuMemCreate/cuMemMap),
// so every bundle is one contiguous range and a freed range is reused
// immediately (best fit, neighbours coalesced).  All users run on the
// context's compute stream, so host-order reuse is stream-ordered reuse.
#pragma once

#include <cuda.h>

#include <cstddef>
#include <map>
#include <vector>

namespace aegis {

class Arena {
 public:
  explicit Arena(int device);
  ~Arena();
  Arena(const Arena&) = delete;
  Arena& operator=(const Arena&) = delete;

  void* alloc(size_t bytes);  // nullptr when physical memory is exhausted
  void free(void* p);
  bool owns(const void* p) const {
    const CUdeviceptr a = (CUdeviceptr)p;
    return base_ && a >= base_ && a < base_ + reserve_;
  }
  size_t mapped() const { return mapped_; }
  size_t in_use() const { return in_use_; }
  size_t largest_free() const;
  void trim();  // unmap whole chunks at the free tail

 private:
  bool grow(size_t need);
  int dev_;
  CUdeviceptr base_ = 0;
  size_t reserve_ = 0, mapped_ = 0, gran_ = 0, in_use_ = 0;
  struct Chunk {
    size_t off, size;
    CUmemGenericAllocationHandle h;
  };
  std::vector<Chunk> chunks_;
  std::map<size_t, size_t> free_;  // offset -> size (inside the mapped prefix)
  std::map<size_t, size_t> used_;  // offset -> size
};

}  // namespace aegis

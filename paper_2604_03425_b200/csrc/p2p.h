// p2p.h -- PCMM reduce-scatter over CUDA IPC / NVLink peer memory (p2p.cu).
#pragma once

#include <vector>

#include "common.cuh"

namespace aegis {

class Context;
constexpr int kP2pHandleBytes = 64;  // sizeof(cudaIpcMemHandle_t)

struct P2pWindow {
  void* own = nullptr;          // this rank's staging window (cudaMalloc, IPC-exported)
  size_t bytes = 0;
  std::vector<void*> peers;     // window of every group rank (peers[self] == own)
  unsigned self = 0;
  ~P2pWindow();
};

P2pWindow* p2p_create(Context& c, size_t bytes, void* handle_out);
void p2p_open(P2pWindow& w, const void* handles, u32 m, u32 self);
void p2p_stage(Context& c, P2pWindow& w, const u64* buf, size_t words);
void p2p_reduce(Context& c, P2pWindow& w, u64* dst, size_t words_per_rank, u32 part);

}  // namespace aegis

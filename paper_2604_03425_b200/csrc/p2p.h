// p2p.h -- PCMM reduce-scatter over CUDA IPC / NVLink peer memory (p2p.cu).
#pragma once

#include <vector>

#include "common.cuh"

namespace aegis {

class Context;
constexpr int kP2pHandleBytes = 64;  // sizeof(cudaIpcMemHandle_t)
constexpr int kP2pMaxPeers = 16;
// window = [flag area][data]; flags (u64): ready[16] | ack[16] | block counters
constexpr size_t kP2pFlagBytes = 4096;
constexpr int kFlagReady = 0, kFlagAck = kP2pMaxPeers, kFlagCount = 2 * kP2pMaxPeers;

struct P2pWindow {
  void* own = nullptr;          // this rank's window (cudaMalloc, IPC-exported): flags + data
  size_t bytes = 0;             // data bytes (after the flag area)
  std::vector<void*> peers;     // window base of every group rank (peers[self] == own)
  unsigned self = 0;
  bool local = false;           // peers are this process's own windows (no IPC mapping)
  u64 epoch = 0;                // exchanges issued through this window (identical on every rank)
  ~P2pWindow();
  __host__ __device__ static u64* flags(void* base) { return static_cast<u64*>(base); }
  __host__ __device__ static u64* data(void* base) { return reinterpret_cast<u64*>(static_cast<char*>(base) + kP2pFlagBytes); }
};

P2pWindow* p2p_create(Context& c, size_t bytes, void* handle_out);
void p2p_open(P2pWindow& w, const void* handles, u32 m, u32 self);
// same-process group (one thread per context, or one thread driving several
// contexts): the peers' windows are used through their device pointers
void p2p_open_local(P2pWindow& w, const std::vector<P2pWindow*>& group, u32 self);
// host-synchronised form (the reduce hook): stage -> barrier -> reduce -> barrier
void p2p_stage(Context& c, P2pWindow& w, const u64* buf, size_t words);
void p2p_reduce(Context& c, P2pWindow& w, u64* dst, size_t words_per_rank, u32 part);
// Device-synchronised reduce-scatter on stream `st` (no host involvement):
// buf holds m shares of `share` words (share q at buf + q*share, uint64 partial
// sums); afterwards buf + self*share holds the uint64 sum over the m ranks.
// Each rank pushes share q into rank q's window (slot self, parity epoch & 1)
// and raises q's ready flag; it then waits for its own m-1 ready flags, sums,
// and acknowledges to every pusher so the slot can be reused two epochs later.
// Every rank of the group must issue the same sequence of exchanges.
void p2p_exchange(P2pWindow& w, u64* buf, size_t share, cudaStream_t st);
// All-gather with the same window protocol: buf holds m shares of `share`
// words; this rank's share (buf + self*share) is pushed to every peer and the
// m-1 others land in place.  Every rank issues the same exchange sequence.
void p2p_allgather(P2pWindow& w, u64* buf, size_t share, cudaStream_t st);
// words of `share` one exchange can carry through this window
size_t p2p_capacity(const P2pWindow& w);

}  // namespace aegis

// p2p.cu -- PCMM reduce-scatter over NVLink peer memory.
//
// When a token group spans m > 1 GPUs, each rank holds uint64 partial sums for
// all of the group's PCMM outputs and must end with the complete sums of the
// lanes it owns (the reference's kReduceOutputs / CombineScatter event,
// comm_plan.hpp:127, 238).  Instead of a library collective every rank
// exposes a window through CUDA IPC (NVLink P2P on a multi-GPU box,
// same-device IPC on a 1-GPU box) and the kernels below move and sum the
// shares directly.
//
// Two forms:
//  * host-synchronised (the reduce hook; kept as the fallback):
//    stage -> group barrier -> p2p_reduce (pull + sum) -> group barrier.
//  * device-synchronised (p2p_exchange, the executor's default when a window
//    is attached): everything is issued on the context's comm stream with
//    CUDA-event edges to the compute stream and flags in the windows --
//      push:  share q of my partials -> window_q.slot[parity][me]; the last
//             block fences (system scope) and raises window_q.ready[me]
//      wait:  one warp spins (ld.acquire.sys) on my ready[r] >= epoch
//      sum:   my share += the m-1 received slots (local HBM reads); the last
//             block raises window_r.ack[me] = epoch at every pusher r
//    A push of epoch e waits for ack >= e - 2 from its target first, so a slot
//    (two parities) is never overwritten before its reader is done.  No host
//    barrier and no Python run inside the layer.
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "context.h"
#include "p2p.h"

namespace aegis {

namespace {

struct PeerPtrs {
  u64* w[kP2pMaxPeers];
};

__device__ __forceinline__ u64 ld_acquire_sys(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(u64* p, u64 v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// dst[i] = sum_r window_r[share_off + i] (uint64), 4 words per thread (256-bit loads)
__global__ void __launch_bounds__(256) p2p_reduce_kernel(const PeerPtrs pw, u32 m, size_t share_off, u64* dst,
                                                          size_t words) {
  const size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i >= words) return;
  u64 s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (u32 r = 0; r < m; ++r) {
    u64 a, b, c, d;
    ld256g(pw.w[r] + share_off + i, a, b, c, d);
    s0 += a;
    s1 += b;
    s2 += c;
    s3 += d;
  }
  st256g(dst + i, s0, s1, s2, s3);
}

__device__ __forceinline__ u64 globaltimer_ns() {
  u64 t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// one warp: wait until flags[base + r] >= target for every r != self.  A peer
// that never arrives (crashed rank, mismatched op sequence) traps after 60 s,
// so the failure surfaces as a CUDA error at aegis_sync instead of a hang.
__global__ void p2p_wait_kernel(const u64* flags, u32 base, u32 m, u32 self, u64 target) {
  const u32 r = threadIdx.x;
  if (r >= m || r == self) return;
  const u64 t0 = globaltimer_ns();
  while (ld_acquire_sys(flags + base + r) < target) {
    __nanosleep(256);
    if (globaltimer_ns() - t0 > 60ull * 1000000000ull) __trap();
  }
}

// Last-block completion: every block fences its writes at system scope and
// counts itself in; the last one stores `value` into flag `field` + self of
// each peer window (release, system scope) and resets the counter.
__device__ void signal_when_done(u64* counter, const PeerPtrs& peers, u32 m, u32 self, u32 field, u64 value) {
  __threadfence_system();  // every thread's stores (local or to peer windows) ordered before the count
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned total = gridDim.x * gridDim.y;
    last = atomicAdd(reinterpret_cast<unsigned long long*>(counter), 1ull) == total - 1;
  }
  __syncthreads();
  if (!last) return;
  if (threadIdx.x < m && threadIdx.x != self) {
    __threadfence_system();
    st_release_sys(P2pWindow::flags(peers.w[threadIdx.x]) + field + self, value);
  }
  if (threadIdx.x == 0) *counter = 0;
}

// blockIdx.y = target rank q: src share q (all-gather: my own share, to every
// peer) -> window_q data slot (parity, self)
template <bool GATHER>
__global__ void __launch_bounds__(256) p2p_push_kernel(const PeerPtrs peers, const u64* src, u32 m, u32 self,
                                                       size_t share, size_t slot_words, u32 parity, u64* counter,
                                                       u64 epoch) {
  const u32 q = blockIdx.y;
  if (q != self) {
    u64* dst = P2pWindow::data(peers.w[q]) + ((size_t)parity * m + self) * slot_words;
    const u64* s = src + (size_t)(GATHER ? self : q) * share;
    for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < share;
         i += (size_t)gridDim.x * blockDim.x * 4) {
      u64 a, b, c, d;
      ld256g(s + i, a, b, c, d);
      st256g(dst + i, a, b, c, d);
    }
  }
  signal_when_done(counter, peers, m, self, kFlagReady, epoch);
}

// my share (in place) += the m-1 slots peers pushed into my window
__global__ void __launch_bounds__(256) p2p_sum_kernel(const PeerPtrs peers, u64* mine, u32 m, u32 self, size_t share,
                                                      size_t slot_words, u32 parity, u64* counter, u64 epoch) {
  const u64* slots = P2pWindow::data(peers.w[self]) + (size_t)parity * m * slot_words;
  for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < share;
       i += (size_t)gridDim.x * blockDim.x * 4) {
    u64 s0, s1, s2, s3;
    ld256g(mine + i, s0, s1, s2, s3);
    for (u32 r = 0; r < m; ++r) {
      if (r == self) continue;
      u64 a, b, c, d;
      ld256g(slots + (size_t)r * slot_words + i, a, b, c, d);
      s0 += a;
      s1 += b;
      s2 += c;
      s3 += d;
    }
    st256g(mine + i, s0, s1, s2, s3);
  }
  signal_when_done(counter, peers, m, self, kFlagAck, epoch);
}

// all-gather receive: share r of buf <- the slot peer r pushed into my window
__global__ void __launch_bounds__(256) p2p_collect_kernel(const PeerPtrs peers, u64* buf, u32 m, u32 self,
                                                          size_t share, size_t slot_words, u32 parity, u64* counter,
                                                          u64 epoch) {
  const u64* slots = P2pWindow::data(peers.w[self]) + (size_t)parity * m * slot_words;
  const u32 r = blockIdx.y;
  if (r != self)
    for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < share;
         i += (size_t)gridDim.x * blockDim.x * 4) {
      u64 a, b, c, d;
      ld256g(slots + (size_t)r * slot_words + i, a, b, c, d);
      st256g(buf + (size_t)r * share + i, a, b, c, d);
    }
  signal_when_done(counter, peers, m, self, kFlagAck, epoch);
}

PeerPtrs peer_ptrs(const P2pWindow& w) {
  PeerPtrs pw;
  std::memset(&pw, 0, sizeof(pw));
  for (size_t r = 0; r < w.peers.size(); ++r) pw.w[r] = static_cast<u64*>(w.peers[r]);
  return pw;
}

}  // namespace

P2pWindow::~P2pWindow() {
  if (!local)
    for (size_t r = 0; r < peers.size(); ++r)
      if (r != self && peers[r]) cudaIpcCloseMemHandle(peers[r]);
  if (own) cudaFree(own);
}

P2pWindow* p2p_create(Context& c, size_t bytes, void* handle_out) {
  auto* w = new P2pWindow;
  w->bytes = (bytes + 255) / 256 * 256;
  cudaError_t e = cudaMalloc(&w->own, kP2pFlagBytes + w->bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    delete w;
    throw Error(AEGIS_EOOM, "p2p window allocation failed");
  }
  AEGIS_CHECK_CUDA(cudaMemset(w->own, 0, kP2pFlagBytes));
  if (handle_out) {
    cudaIpcMemHandle_t h;
    AEGIS_CHECK_CUDA(cudaIpcGetMemHandle(&h, w->own));
    static_assert(sizeof(h) == kP2pHandleBytes, "IPC handle size");
    std::memcpy(handle_out, &h, sizeof(h));
  }
  (void)c;
  return w;
}

void p2p_open(P2pWindow& w, const void* handles, u32 m, u32 self) {
  if (m == 0 || m > (u32)kP2pMaxPeers || self >= m) throw Error(AEGIS_EINVAL, "p2p_open: bad group size / rank");
  w.peers.assign(m, nullptr);
  w.self = self;
  w.local = false;
  w.epoch = 0;
  for (u32 r = 0; r < m; ++r) {
    if (r == self) {
      w.peers[r] = w.own;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + (size_t)r * kP2pHandleBytes, sizeof(h));
    void* p = nullptr;
    AEGIS_CHECK_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    w.peers[r] = p;
  }
}

void p2p_open_local(P2pWindow& w, const std::vector<P2pWindow*>& group, u32 self) {
  const u32 m = (u32)group.size();
  if (m == 0 || m > (u32)kP2pMaxPeers || self >= m || group[self] != &w)
    throw Error(AEGIS_EINVAL, "p2p_open_local: bad group / rank");
  w.peers.assign(m, nullptr);
  for (u32 r = 0; r < m; ++r) {
    if (!group[r] || group[r]->bytes != w.bytes) throw Error(AEGIS_EINVAL, "p2p_open_local: windows differ in size");
    w.peers[r] = group[r]->own;
  }
  w.self = self;
  w.local = true;
  w.epoch = 0;
}

size_t p2p_capacity(const P2pWindow& w) {
  const size_t m = std::max<size_t>(1, w.peers.size());
  return (w.bytes / 8) / (2 * m) / 4 * 4;
}

void p2p_stage(Context& c, P2pWindow& w, const u64* buf, size_t words) {
  if (words * 8 > w.bytes) throw Error(AEGIS_EINVAL, "p2p_stage: payload larger than the window");
  AEGIS_CHECK_CUDA(cudaMemcpyAsync(P2pWindow::data(w.own), buf, words * 8, cudaMemcpyDeviceToDevice, c.stream));
  AEGIS_CHECK_CUDA(cudaStreamSynchronize(c.stream));
}

void p2p_reduce(Context& c, P2pWindow& w, u64* dst, size_t words_per_rank, u32 part) {
  const u32 m = (u32)w.peers.size();
  if (!m) throw Error(AEGIS_ELOGIC, "p2p_reduce: window not opened");
  if ((size_t)(part + 1) * words_per_rank * 8 > w.bytes) throw Error(AEGIS_EINVAL, "p2p_reduce: share out of window");
  if (words_per_rank % 4 || reinterpret_cast<uintptr_t>(dst) % 32)
    throw Error(AEGIS_EINVAL, "p2p_reduce: share must be 32-byte aligned whole 4-word groups");
  PeerPtrs pw;
  std::memset(&pw, 0, sizeof(pw));
  for (u32 r = 0; r < m; ++r) pw.w[r] = P2pWindow::data(w.peers[r]);
  const size_t threads = words_per_rank / 4;
  if (threads) {
    p2p_reduce_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, c.stream>>>(pw, m, (size_t)part * words_per_rank,
                                                                              dst, words_per_rank);
    AEGIS_CHECK_CUDA(cudaGetLastError());
    c.count();
  }
  AEGIS_CHECK_CUDA(cudaStreamSynchronize(c.stream));
}

void p2p_exchange(P2pWindow& w, u64* buf, size_t share, cudaStream_t st) {
  const u32 m = (u32)w.peers.size();
  if (m < 2) throw Error(AEGIS_ELOGIC, "p2p_exchange: window not opened for a group");
  if (share % 4 || reinterpret_cast<uintptr_t>(buf) % 32)
    throw Error(AEGIS_EINVAL, "p2p_exchange: shares must be 32-byte aligned whole 4-word groups");
  const size_t slot = p2p_capacity(w);
  if (share > slot) throw Error(AEGIS_EINVAL, "p2p_exchange: share larger than the window slot");
  const u64 e = ++w.epoch;
  const u32 parity = (u32)(e & 1);
  const PeerPtrs pw = peer_ptrs(w);
  u64* fl = P2pWindow::flags(w.own);
  // the slot (parity) this push overwrites was last read at epoch e - 2
  if (e > 2) p2p_wait_kernel<<<1, 32, 0, st>>>(fl, kFlagAck, m, w.self, e - 2);
  const unsigned bx = (unsigned)std::min<size_t>(256, std::max<size_t>(1, share / 1024));
  p2p_push_kernel<false><<<dim3(bx, m), 256, 0, st>>>(pw, buf, m, w.self, share, slot, parity, fl + kFlagCount, e);
  p2p_wait_kernel<<<1, 32, 0, st>>>(fl, kFlagReady, m, w.self, e);
  p2p_sum_kernel<<<bx, 256, 0, st>>>(pw, buf + (size_t)w.self * share, m, w.self, share, slot, parity,
                                     fl + kFlagCount + 1, e);
  AEGIS_CHECK_CUDA(cudaGetLastError());
}

void p2p_allgather(P2pWindow& w, u64* buf, size_t share, cudaStream_t st) {
  const u32 m = (u32)w.peers.size();
  if (m < 2) throw Error(AEGIS_ELOGIC, "p2p_allgather: window not opened for a group");
  if (share % 4 || reinterpret_cast<uintptr_t>(buf) % 32)
    throw Error(AEGIS_EINVAL, "p2p_allgather: shares must be 32-byte aligned whole 4-word groups");
  const size_t slot = p2p_capacity(w);
  if (share > slot) throw Error(AEGIS_EINVAL, "p2p_allgather: share larger than the window slot");
  const u64 e = ++w.epoch;
  const u32 parity = (u32)(e & 1);
  const PeerPtrs pw = peer_ptrs(w);
  u64* fl = P2pWindow::flags(w.own);
  if (e > 2) p2p_wait_kernel<<<1, 32, 0, st>>>(fl, kFlagAck, m, w.self, e - 2);
  const unsigned bx = (unsigned)std::min<size_t>(256, std::max<size_t>(1, share / 1024));
  p2p_push_kernel<true><<<dim3(bx, m), 256, 0, st>>>(pw, buf, m, w.self, share, slot, parity, fl + kFlagCount, e);
  p2p_wait_kernel<<<1, 32, 0, st>>>(fl, kFlagReady, m, w.self, e);
  p2p_collect_kernel<<<dim3(bx, m), 256, 0, st>>>(pw, buf, m, w.self, share, slot, parity, fl + kFlagCount + 1, e);
  AEGIS_CHECK_CUDA(cudaGetLastError());
}

}  // namespace aegis

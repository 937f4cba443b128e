// p2p.cu -- PCMM reduce-scatter over NVLink peer memory.
//
// When a token group spans m > 1 GPUs, each rank holds uint64 partial sums for
// all of the group's PCMM outputs and must end with the complete sums of the
// lanes it owns (the reference's kReduceOutputs, comm_plan.hpp:127, 238).
// Instead of a library collective, every rank exposes a staging window through
// CUDA IPC; after the group barrier each rank's kernel reads its share straight
// out of the m windows (NVLink P2P loads; same-device IPC on a 1-GPU box),
// sums them (uint64: the ncclUint64-sum semantics of the executor's reduce
// hook) and writes them over its own share; the executor's reduce_lanes pass
// then canonicalises (residues < 2^46, so m * p never wraps).
//
//   aegis_p2p_create   window of `bytes`, exports its 64-byte IPC handle
//   aegis_p2p_open     maps the m handles of the group (own window stays local)
//   aegis_p2p_stage    partial sums -> own window (stream-ordered, synchronous)
//   aegis_p2p_reduce   dst lanes = sum over the m windows of this rank's share
// The host runs stage -> group barrier -> reduce -> group barrier.
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "context.h"
#include "p2p.h"

namespace aegis {

namespace {

constexpr int kMaxPeers = 16;
struct PeerPtrs {
  const u64* w[kMaxPeers];
};

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

}  // namespace

P2pWindow::~P2pWindow() {
  for (size_t r = 0; r < peers.size(); ++r)
    if (r != self && peers[r]) cudaIpcCloseMemHandle(peers[r]);
  if (own) cudaFree(own);
}

P2pWindow* p2p_create(Context& c, size_t bytes, void* handle_out) {
  auto* w = new P2pWindow;
  w->bytes = bytes;
  cudaError_t e = cudaMalloc(&w->own, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    delete w;
    throw Error(AEGIS_EOOM, "p2p window allocation failed");
  }
  cudaIpcMemHandle_t h;
  AEGIS_CHECK_CUDA(cudaIpcGetMemHandle(&h, w->own));
  static_assert(sizeof(h) == kP2pHandleBytes, "IPC handle size");
  std::memcpy(handle_out, &h, sizeof(h));
  (void)c;
  return w;
}

void p2p_open(P2pWindow& w, const void* handles, u32 m, u32 self) {
  if (m == 0 || m > (u32)kMaxPeers || self >= m) throw Error(AEGIS_EINVAL, "p2p_open: bad group size / rank");
  w.peers.assign(m, nullptr);
  w.self = self;
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

void p2p_stage(Context& c, P2pWindow& w, const u64* buf, size_t words) {
  if (words * 8 > w.bytes) throw Error(AEGIS_EINVAL, "p2p_stage: payload larger than the window");
  AEGIS_CHECK_CUDA(cudaMemcpyAsync(w.own, buf, words * 8, cudaMemcpyDeviceToDevice, c.stream));
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
  for (u32 r = 0; r < m; ++r) pw.w[r] = static_cast<const u64*>(w.peers[r]);
  const size_t threads = words_per_rank / 4;
  if (threads) {
    p2p_reduce_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, c.stream>>>(pw, m, (size_t)part * words_per_rank,
                                                                              dst, words_per_rank);
    AEGIS_CHECK_CUDA(cudaGetLastError());
    c.count();
  }
  AEGIS_CHECK_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace aegis

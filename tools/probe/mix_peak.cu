// Mixed-pipe butterfly probe (sm_100a): warps w % 8 < K run integer Shoup
// butterflies (IMAD pipe), the others exact FP64 butterflies (DFMA pipe), in
// the same CTA.  Prints total butterflies per SM clock for K = 0..8, i.e. how
// much an INT/FP64 split of an NTT's butterflies could raise throughput over
// the FP64-only form (K = 0).  Clock: clock64() cycles of block 0 / elapsed.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ void body_int(u64 (&x)[8], u64 w, u64 wp, u64 p) {
  const u64 two_p = 2 * p;
#pragma unroll
  for (int h = 4; h >= 1; h >>= 1)
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      if (v & h) continue;
      u64 q = __umul64hi(x[v + h], wp);
      u64 t = x[v + h] * w - q * p;
      u64 a = x[v];
      a = a >= two_p ? a - two_p : a;  // Harvey lazy range [0, 2p)
      x[v] = a + t;
      x[v + h] = a + two_p - t;
    }
}
__device__ __forceinline__ void body_f64(double (&x)[8], double w, double wp, double p) {
  const double M = 6755399441055744.0;
#pragma unroll
  for (int h = 4; h >= 1; h >>= 1)
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      if (v & h) continue;
      const double y = x[v + h];
      const double hh = y * w;
      const double l = fma(y, w, -hh);
      const double q = fma(y, wp, M) - M;
      const double r = fma(-q, p, hh) + l;
      const double a = x[v];
      x[v] = a + r;
      x[v + h] = a - r;
    }
}
__global__ void mix(u64* out, long long* cyc, int iters, int k_int, u64 w, u64 wp, u64 p, double wd, double wpd,
                    double pd) {
  const long long t0 = clock64();
  const int warp = threadIdx.x >> 5;
  u64 s = 0;
  if ((warp & 7) < k_int) {
    u64 x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 7 + i;
    for (int it = 0; it < iters; ++it) body_int(x, w, wp, p);
    for (int i = 0; i < 8; ++i) s += x[i];
  } else {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 7 + i;
    for (int it = 0; it < iters; ++it) body_f64(x, wd, wpd, pd);
    for (int i = 0; i < 8; ++i) s += (u64)(long long)x[i];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = clock64() - t0;
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 3, threads = 256, iters = 4096;
  u64* buf;
  long long* cyc;
  cudaMalloc(&buf, (size_t)blocks * threads * 8);
  cudaMalloc(&cyc, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double nb = (double)blocks * threads * iters * 12;
  const u64 p = (1ULL << 45) + 0x1234567ULL * 2 + 1;
  const u64 w = 123456789;
  const u64 wp = (u64)(((unsigned __int128)w << 64) / p);
  for (int rep = 0; rep < 2; ++rep)
    for (int k = 0; k <= 8; ++k) {
      float ms;
      cudaEventRecord(e0);
      mix<<<blocks, threads>>>(buf, cyc, iters, k, w, wp, p, (double)w, (double)w / p, (double)p);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      long long c = 0;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double clk = c / (ms * 1e-3);  // cycles of block 0 over the launch (close to SM clock)
      if (rep == 1)
        printf("int_warps=%d/8  %.3f ms  clk~%.0f MHz  %.2f bfly/clk/SM\n", k, ms, clk / 1e6,
               nb / (ms * 1e-3) / sms / clk);
    }
  return 0;
}

// Butterfly throughput probe on sm_100a: integer Shoup (lazy) vs FP64 vs hybrid.
// Each thread runs independent radix-2 butterflies on 8 register values.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__global__ void bfly_int(u64* out, int iters, u64 w, u64 wp, u64 p) {
  u64 x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 7 + i;
  const u64 two_p = 2 * p;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int h = 4; h >= 1; h >>= 1)
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        if (v & h) continue;
        u64 q = __umul64hi(x[v + h], wp);
        u64 t = x[v + h] * w - q * p;
        u64 a = x[v];
        x[v] = a + t; x[v + h] = a + two_p - t;
        x[v] -= (x[v] >= (u64)1 << 53) ? (u64)1 << 52 : 0;  // keep bounded (cheap)
        x[v + h] &= ((u64)1 << 53) - 1;
      }
  }
  u64 s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void bfly_f64(double* out, int iters, double w, double wp, double p) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 7 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int h = 4; h >= 1; h >>= 1)
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        if (v & h) continue;
        const double y = x[v + h];
        const double hh = y * w;
        const double l = fma(y, w, -hh);
        const double q = rint(y * wp);
        double r = fma(-q, p, hh);
        r += l;
        const double a = x[v];
        x[v] = a + r; x[v + h] = a - r;
      }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void bfly_f64_magic(double* out, int iters, double w, double wp, double p) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 7 + i;
  const double M = 6755399441055744.0;  // 1.5 * 2^52
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int h = 4; h >= 1; h >>= 1)
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        if (v & h) continue;
        const double y = x[v + h];
        const double hh = y * w;
        const double l = fma(y, w, -hh);
        const double q = fma(y, wp, M) - M;
        double r = fma(-q, p, hh);
        r += l;
        const double a = x[v];
        x[v] = a + r; x[v + h] = a - r;
      }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 2048;
  void* buf; cudaMalloc(&buf, (size_t)blocks * threads * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double nb = (double)blocks * threads * iters * 12;  // 12 butterflies per iteration
  const u64 p = (1ULL << 45) + 1; const u64 w = 123456789; const u64 wp = (u64)(((unsigned __int128)w << 64) / p);
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0); bfly_int<<<blocks, threads>>>((u64*)buf, iters, w, wp, p); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("int-shoup : %.3f ms  %.2f bfly/clk/SM\n", ms, nb / (ms * 1e-3) / sms / 1.965e9);
    cudaEventRecord(e0); bfly_f64<<<blocks, threads>>>((double*)buf, iters, (double)w, (double)w / p, (double)p); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("f64-rint  : %.3f ms  %.2f bfly/clk/SM\n", ms, nb / (ms * 1e-3) / sms / 1.965e9);
    cudaEventRecord(e0); bfly_f64_magic<<<blocks, threads>>>((double*)buf, iters, (double)w, (double)w / p, (double)p); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("f64-magic : %.3f ms  %.2f bfly/clk/SM\n", ms, nb / (ms * 1e-3) / sms / 1.965e9);
  }
  return 0;
}

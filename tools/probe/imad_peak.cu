// Integer-pipe microbenchmark: 32-bit IMAD peak and 64-bit Shoup modmul rate on sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void imad32(uint32_t* out, int iters, uint32_t a, uint32_t b) {
  uint32_t x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
      x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 ^ x1 ^ x2 ^ x3 ^ x4 ^ x5 ^ x6 ^ x7;
}
__device__ __forceinline__ uint64_t shoup(uint64_t y, uint64_t w, uint64_t wp, uint64_t p) {
  uint64_t q = __umul64hi(y, wp);
  return y * w - q * p;
}
__global__ void shoup64(uint64_t* out, int iters, uint64_t w, uint64_t wp, uint64_t p) {
  uint64_t x0 = threadIdx.x, x1 = x0 + 11, x2 = x0 + 22, x3 = x0 + 33;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = shoup(x0, w, wp, p); x1 = shoup(x1, w, wp, p); x2 = shoup(x2, w, wp, p); x3 = shoup(x3, w, wp, p);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 ^ x1 ^ x2 ^ x3;
}
__global__ void dfma(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * 8, threads = 256, iters = 4096;
  void* buf; cudaMalloc(&buf, (size_t)blocks * threads * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); imad32<<<blocks, threads>>>((uint32_t*)buf, iters, 1664525u, 1013904223u); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * iters * 16 * 8;
    printf("imad32: %.3f ms  %.2f Tops/s (%.1f per SM per clk @1.965GHz)\n", ms, ops / ms / 1e9, ops / (ms * 1e-3) / sms / 1.965e9);
    cudaEventRecord(e0); shoup64<<<blocks, threads>>>((uint64_t*)buf, iters, 12345, 0x123456789abcdefULL, (1ULL << 49) + 1); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    ops = (double)blocks * threads * iters * 16 * 4;
    printf("shoup64: %.3f ms  %.2f Tmodmul/s (%.2f per SM per clk)\n", ms, ops / ms / 1e9, ops / (ms * 1e-3) / sms / 1.965e9);
    cudaEventRecord(e0); dfma<<<blocks, threads>>>((double*)buf, iters, 0.999, 1e-3); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    ops = (double)blocks * threads * iters * 16 * 8;
    printf("dfma: %.3f ms  %.2f Tfma/s (%.1f per SM per clk)\n", ms, ops / ms / 1e9, ops / (ms * 1e-3) / sms / 1.965e9);
  }
  printf("sms=%d\n", sms);
  return 0;
}

// FP64 FMA throughput probe (independent chains), and smem 16-B bandwidth probe.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k_fma(double *out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __fma_rn(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1.2345) out[0] = s;
}
template <int CH>
__global__ void k_mul(double *out, int iters, double a) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __dmul_rn(x[c], a);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double *o;
  cudaMalloc(&o, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int dev;
  cudaGetDevice(&dev);
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  for (int threads : {256, 512, 1024}) {
    for (int blocks_per_sm : {1, 2, 4}) {
      const int iters = 4096;
      k_fma<8><<<sms * blocks_per_sm, threads>>>(o, 16, 1.0000001, 1e-9);
      cudaEventRecord(a);
      k_fma<8><<<sms * blocks_per_sm, threads>>>(o, iters, 1.0000001, 1e-9);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double fmas = (double)sms * blocks_per_sm * threads * iters * 8;
      printf("DFMA threads=%4d blk/SM=%d: %.2f TFMA/s = %.1f TFLOP/s  (%.1f FMA/clk/SM at %d MHz nominal)\n",
             threads, blocks_per_sm, fmas / ms / 1e9, 2 * fmas / ms / 1e9, fmas / (ms * 1e-3) / sms / (clk * 1e3),
             clk / 1000);
    }
  }
  const int iters = 4096;
  cudaEventRecord(a);
  k_mul<8><<<sms * 2, 1024>>>(o, iters, 1.0000001);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("DMUL: %.2f T/s\n", (double)sms * 2 * 1024 * iters * 8 / ms / 1e9);
  return 0;
}

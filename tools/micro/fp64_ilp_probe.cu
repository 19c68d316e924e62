// FP64 pipe probe: DFMA throughput per SM as a function of resident warps per scheduler and of
// the independent chains per thread (ILP), and the same for the DMUL -> DFMA pairs of a complex
// multiply.  Answers: how many warps x how much ILP saturate the FP64 pipe of one SM sub-partition?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_ilp_probe fp64_ilp_probe.cu
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
// complex multiply chains: CH amplitudes, each re/im: 2 DMUL then 2 DFMA (depth 2 per step)
template <int CH>
__global__ void k_cmul(double *out, int iters, double qr, double qi) {
  double xr[CH], xi[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) xr[c] = threadIdx.x * 1e-3 + c, xi[c] = 0.5 + c;
  for (int i = 0; i < iters; ++i) {
    double tr[CH], ti[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) tr[c] = __dmul_rn(xi[c], qi), ti[c] = __dmul_rn(xr[c], qi);
#pragma unroll
    for (int c = 0; c < CH; ++c) xr[c] = __fma_rn(qr, xr[c], -tr[c]), xi[c] = __fma_rn(qr, xi[c], ti[c]);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += xr[c] + xi[c];
  if (s == 1.2345) out[0] = s;
}
template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}
int main() {
  double *o;
  cudaMalloc(&o, 8);
  int dev, sms;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int iters = 2048;
  printf("ops per clock per SM at 1.9 GHz nominal would be 64; T ops/s = total DFMA-class instructions x 32 lanes\n");
  for (int wps : {1, 2, 3, 4, 6, 8}) {  // warps per scheduler (4 schedulers per SM)
    const int threads = wps * 4 * 32;
    float m1 = timeit([&] { k_fma<1><<<sms, threads>>>(o, iters, 1.0000001, 1e-9); });
    float m2 = timeit([&] { k_fma<2><<<sms, threads>>>(o, iters, 1.0000001, 1e-9); });
    float m4 = timeit([&] { k_fma<4><<<sms, threads>>>(o, iters, 1.0000001, 1e-9); });
    float m8 = timeit([&] { k_fma<8><<<sms, threads>>>(o, iters, 1.0000001, 1e-9); });
    float m16 = timeit([&] { k_fma<16><<<sms, threads>>>(o, iters, 1.0000001, 1e-9); });
    auto r = [&](float ms, int ch) { return (double)sms * threads * iters * ch / ms / 1e9; };
    printf("DFMA warps/sched=%d: ILP1 %.2f  ILP2 %.2f  ILP4 %.2f  ILP8 %.2f  ILP16 %.2f  T/s\n", wps, r(m1, 1), r(m2, 2),
           r(m4, 4), r(m8, 8), r(m16, 16));
    float c1 = timeit([&] { k_cmul<1><<<sms, threads>>>(o, iters, 0.7, 0.7); });
    float c2 = timeit([&] { k_cmul<2><<<sms, threads>>>(o, iters, 0.7, 0.7); });
    float c4 = timeit([&] { k_cmul<4><<<sms, threads>>>(o, iters, 0.7, 0.7); });
    float c8 = timeit([&] { k_cmul<8><<<sms, threads>>>(o, iters, 0.7, 0.7); });
    auto rc = [&](float ms, int ch) { return (double)sms * threads * iters * ch * 4 / ms / 1e9; };
    printf("CMUL warps/sched=%d: 1 amp %.2f  2 amps %.2f  4 amps %.2f  8 amps %.2f  T/s\n", wps, rc(c1, 1), rc(c2, 2),
           rc(c4, 4), rc(c8, 8));
  }
  return 0;
}

// Microbenchmark: variants of the single-qubit pair kernel (block size, unroll, cache hints,
// grid-stride persistence) and controlled c=0 with half-sector writes.
#include <functional>
#include "../../paper_1601_07195_b200/csrc/svb200.cu"

template <int B, int U, int HINT>
__global__ void __launch_bounds__(B) v_pairs(double2 *__restrict__ a, uint64_t npairs, int tv, GateQ q) {
  const uint64_t tb = 1ull << tv;
  const uint64_t p0 = (uint64_t)blockIdx.x * (B * U) + threadIdx.x;
  double2 x0[U], x1[U];
  uint64_t i0[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t p = p0 + (uint64_t)u * B;
    i0[u] = insert_zero(p, tv);
    if (HINT == 1) { x0[u] = __ldcs(a + i0[u]); x1[u] = __ldcs(a + i0[u] + tb); }
    else if (HINT == 2) { x0[u] = __ldlu(a + i0[u]); x1[u] = __ldlu(a + i0[u] + tb); }
    else { x0[u] = a[i0[u]]; x1[u] = a[i0[u] + tb]; }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    double2 n0 = mix(x0[u], x1[u], q.v[0], q.v[1], q.v[2], q.v[3]);
    double2 n1 = mix(x0[u], x1[u], q.v[4], q.v[5], q.v[6], q.v[7]);
    if (HINT >= 1) { __stcs(a + i0[u], n0); __stcs(a + i0[u] + tb, n1); }
    else { a[i0[u]] = n0; a[i0[u] + tb] = n1; }
  }
}

// persistent grid-stride with one-batch lookahead
template <int B, int U>
__global__ void __launch_bounds__(B) v_persist(double2 *__restrict__ a, uint64_t npairs, int tv, GateQ q) {
  const uint64_t tb = 1ull << tv;
  const uint64_t stride = (uint64_t)gridDim.x * B * U;
  for (uint64_t base = (uint64_t)blockIdx.x * (B * U) + threadIdx.x; base < npairs; base += stride) {
    double2 x0[U], x1[U];
    uint64_t i0[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      i0[u] = insert_zero(base + (uint64_t)u * B, tv);
      x0[u] = a[i0[u]];
      x1[u] = a[i0[u] + tb];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a[i0[u]] = mix(x0[u], x1[u], q.v[0], q.v[1], q.v[2], q.v[3]);
      a[i0[u] + tb] = mix(x0[u], x1[u], q.v[4], q.v[5], q.v[6], q.v[7]);
    }
  }
}

__global__ void v_copy(const double2 *__restrict__ s, double2 *__restrict__ d, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    d[i] = s[i];
}
__global__ void v_read(const double2 *__restrict__ s, uint64_t n, double *out) {
  double acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    acc += s[i].x;
  if (acc == 1.2345) out[0] = acc;
}

static float time_ms(std::function<void()> f, int reps = 7) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  return best;
}

#define RUN(NAME, B, U, H)                                                                              \
  {                                                                                                     \
    float ms = time_ms([&] { v_pairs<B, U, H><<<(unsigned)(np / (B * U)), B>>>(a, np, tv, q); });       \
    printf("%-28s k=%2d %.3f ms %.0f GB/s\n", NAME, tv, ms, bytes / ms / 1e6);                          \
  }

int main() {
  const int m = 30;
  const uint64_t n = 1ull << m, np = n >> 1;
  const double bytes = 32.0 * n;
  double2 *a, *b;
  double *o;
  cudaMalloc(&a, sizeof(double2) * n);
  cudaMalloc(&b, sizeof(double2) * n);
  cudaMalloc(&o, 8);
  cudaMemset(a, 0, sizeof(double2) * n);
  GateQ q = {{0.6, 0.0, 0.8, 0.0, 0.8, 0.0, -0.6, 0.0}};
  int sms = 148;
  for (int tv : {5, 12, 29}) {
    RUN("B256 U4", 256, 4, 0);
    RUN("B256 U2", 256, 2, 0);
    RUN("B256 U8", 256, 8, 0);
    RUN("B128 U4", 128, 4, 0);
    RUN("B512 U2", 512, 2, 0);
    RUN("B256 U4 ldcs/stcs", 256, 4, 1);
    RUN("B256 U4 ldlu/stcs", 256, 4, 2);
    for (int mult : {4, 8, 16}) {
      float ms = time_ms([&] { v_persist<256, 4><<<sms * mult, 256>>>(a, np, tv, q); });
      printf("persist x%-2d                  k=%2d %.3f ms %.0f GB/s\n", mult, tv, ms, bytes / ms / 1e6);
    }
  }
  float ms = time_ms([&] { v_copy<<<sms * 16, 256>>>(a, b, n); });
  printf("copy 16GiB->16GiB %.3f ms %.0f GB/s (r+w)\n", ms, 2.0 * 16 * n / ms / 1e6);
  ms = time_ms([&] { cudaMemcpyAsync(b, a, 16 * n, cudaMemcpyDeviceToDevice); });
  printf("cudaMemcpy D2D   %.3f ms %.0f GB/s (r+w)\n", ms, 2.0 * 16 * n / ms / 1e6);
  ms = time_ms([&] { v_read<<<sms * 16, 256>>>(a, n, o); });
  printf("read-only        %.3f ms %.0f GB/s\n", ms, 16.0 * n / ms / 1e6);
  // controlled c=0: virtual-map (half-sector writes) vs predicated full stream
  double qq[8] = {0.6, 0.0, 0.8, 0.0, 0.8, 0.0, -0.6, 0.0};
  for (int t : {1, 7, 29}) {
    float m1 = time_ms([&] { launch_local<MODE_CTL>(a, m - 1, t - 1, 0, load_q(qq), 0, "ctl"); });
    float m2 = time_ms([&] { sv_apply_controlled(a, m, 0, t, qq, 0); });
    printf("c=0 t=%2d virtual %.3f ms (%.0f acct)  pred %.3f ms (%.0f acct)\n", t, m1, 16.0 * n / m1 / 1e6, m2,
           16.0 * n / m2 / 1e6);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}

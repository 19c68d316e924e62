// Microbenchmark: controlled gate with low control bit under different L2 fetch granularities.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include -o /tmp/ctl_probe tools/micro/ctl_probe.cu
#include <functional>
#include "../../paper_1601_07195_b200/csrc/svb200.cu"

static float time_ms(std::function<void()> f, int reps) {
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

int main() {
  const int m = 30;
  double2 *a;
  cudaMalloc(&a, sizeof(double2) << m);
  cudaMemset(a, 0, sizeof(double2) << m);
  double q[8] = {0.6, 0.0, 0.8, 0.0, 0.8, 0.0, -0.6, 0.0};
  for (int gran : {128, 64, 32}) {
    cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
    size_t got = 0;
    cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
    printf("fetch granularity request %d -> %zu (%s)\n", gran, got, cudaGetErrorString(e));
    for (int c : {0, 1, 2, 3, 4, 8}) {
      for (int t : {0, 7, 29}) {
        if (c == t) continue;
        float ms = time_ms([&] { sv_apply_controlled(a, m, c, t, q, 0); }, 5);
        // predicated full-stream variant for comparison
        const int tv = t;
        float ms2 = time_ms([&] { launch_local<MODE_PRED>(a, m, tv, c, load_q(q), 0, "pred"); }, 5);
        printf("  c=%2d t=%2d ctl %.3f ms (%.0f GB/s acct)   pred %.3f ms (%.0f GB/s acct)\n", c, t, ms,
               (16.0 * (1ull << m)) / ms / 1e6, ms2, (16.0 * (1ull << m)) / ms2 / 1e6);
      }
    }
    float ms = time_ms([&] { sv_apply_single(a, m, 9, q, 0); }, 5);
    printf("  single k=9 %.3f ms (%.0f GB/s)\n", ms, (32.0 * (1ull << m)) / ms / 1e6);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

// Launch cost vs kernel-parameter size on this GPU: back-to-back launches of an
// (almost) empty kernel taking a __grid_constant__ struct of S bytes, timed with
// CUDA events (device time per launch) and wall clock (host time per launch).
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>

template <int S>
struct P {
  unsigned long long w[S / 8];
};

template <int S>
__global__ void k(const __grid_constant__ P<S> p, unsigned long long* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && p.w[S / 8 - 1] == 12345) *out = p.w[0];
}

template <int S>
void run(unsigned long long* d, int grid, bool coop) {
  P<S> p{};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = coop ? 1 : 0;
  for (int i = 0; i < 100; ++i) cudaLaunchKernelEx(&cfg, k<S>, p, d);
  cudaDeviceSynchronize();
  const int n = 2000;
  auto t0 = std::chrono::steady_clock::now();
  cudaEventRecord(a);
  for (int i = 0; i < n; ++i) cudaLaunchKernelEx(&cfg, k<S>, p, d);
  cudaEventRecord(b);
  auto t1 = std::chrono::steady_clock::now();
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  printf("{\"param_bytes\": %d, \"grid\": %d, \"cooperative\": %d, \"device_us_per_launch\": %.3f, \"host_us_per_launch\": %.3f}\n",
         S, grid, (int)coop, ms * 1e3 / n, std::chrono::duration<double, std::micro>(t1 - t0).count() / n);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  for (int coop = 0; coop < 2; ++coop)
    for (int grid : {1, 148, 592}) {
      run<256>(d, grid, coop);
      run<4096>(d, grid, coop);
      run<12288>(d, grid, coop);
      run<30720>(d, grid, coop);
    }
  return 0;
}

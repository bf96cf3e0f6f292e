// Launch-to-launch gap on one stream as a function of the kernel-parameter size, the
// cooperative attribute and the dynamic shared memory: 200 back-to-back launches of a
// kernel that spins for `spin_ns` (globaltimer) on 128 CTAs x 288 threads; the gap is
// (period - spin) per launch, from CUDA events.  The fused ring kernel takes a 14.6 KB
// FusedParams by value; this says what that costs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/launch_gap_probe tools/launch_gap_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

template <int BYTES>
struct Blob {
  unsigned long long spin_ns;
  unsigned long long* sink;
  char pad[BYTES - 16];
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <int BYTES>
__global__ void spin_kernel(const Blob<BYTES> p) {

  const unsigned long long t0 = gtimer();
  if (p.spin_ns)
    while (gtimer() - t0 < p.spin_ns) {
    }
  if (threadIdx.x == 0 && blockIdx.x == 0) p.sink[0] = t0 + p.pad[BYTES - 17];
}

template <int BYTES>
float run(int coop, size_t smem, unsigned long long spin_ns, unsigned long long* sink) {
  Blob<BYTES> p = {};
  p.spin_ns = spin_ns;
  p.sink = sink;
  CK(cudaFuncSetAttribute(spin_kernel<BYTES>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(128);
  cfg.blockDim = dim3(288);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = 0;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = coop ? 1 : 0;
  for (int i = 0; i < 20; ++i) CK(cudaLaunchKernelEx(&cfg, spin_kernel<BYTES>, p));
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int iters = 200;
  CK(cudaEventRecord(e0));
  for (int i = 0; i < iters; ++i) CK(cudaLaunchKernelEx(&cfg, spin_kernel<BYTES>, p));
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  return ms * 1e3f / iters;  // us per launch
}

int main() {
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 64));
  printf("[\n");
  bool first = true;
  for (unsigned long long spin : {0ull, 100000ull})
    for (int coop = 0; coop < 2; ++coop)
      for (size_t smem : {(size_t)0, (size_t)(100 << 10)}) {
        const float a = run<64>(coop, smem, spin, sink);
        const float b = run<4096>(coop, smem, spin, sink);
        const float c = run<8192>(coop, smem, spin, sink);
        const float d = run<14656>(coop, smem, spin, sink);
        const float e = run<30000>(coop, smem, spin, sink);
        const float s = spin / 1000.0f;
        printf("%s{\"spin_us\": %.0f, \"cooperative\": %d, \"smem\": %zu, \"us_per_launch\": {\"64\": %.2f, "
               "\"4096\": %.2f, \"8192\": %.2f, \"14656\": %.2f, \"30000\": %.2f}, \"gap_us\": {\"64\": %.2f, "
               "\"4096\": %.2f, \"8192\": %.2f, \"14656\": %.2f, \"30000\": %.2f}}",
               first ? "" : ",\n", s, coop, smem, a, b, c, d, e, a - s, b - s, c - s, d - s, e - s);
        first = false;
      }
  printf("\n]\n");
  return 0;
}

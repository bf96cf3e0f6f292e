// How long does a system-scope fence take on an SM that keeps pushing data to
// a peer GPU over NVLink?  (Tuning probe for the ring kernel's signalling.)
//
// Each CTA: `pushers` warps stream `bytes_per_cta` into the peer (SM stores or
// TMA bulk stores from shared memory); one prober warp repeatedly executes
//   mode 0: fence.acq_rel.sys
//   mode 1: cp.async.bulk.wait_group (TMA pushes are issued by the prober itself;
//           it waits for the group issued `lag` groups earlier, then fences)
// and records the latency with %globaltimer.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fence_probe tools/fence_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e = (x);                                                                 \
    if (e != cudaSuccess) {                                                              \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);     \
      exit(1);                                                                           \
    }                                                                                    \
  } while (0)

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void probe_stores_v2(char* dst, size_t per_cta, unsigned long long* lat, int nprobe) {
  // pusher warps stream stores to the peer; the prober warp fences and times it
  const int pushers = (blockDim.x / 32) - 1;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  char* base = dst + blockIdx.x * per_cta;
  if (warp < pushers) {
    const size_t n = per_cta / 16;
    for (size_t i = warp * 32 + lane; i < n; i += pushers * 32) {
      uint4 v = make_uint4(i, i, i, i);
      *reinterpret_cast<uint4*>(base + i * 16) = v;
    }
  } else if (lane == 0) {
    unsigned long long sum = 0, mx = 0;
    for (int p = 0; p < nprobe; ++p) {
      unsigned long long t0 = gt();
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      unsigned long long d = gt() - t0;
      sum += d;
      mx = d > mx ? d : mx;
      __nanosleep(2000);
    }
    lat[blockIdx.x * 2] = sum / nprobe;
    lat[blockIdx.x * 2 + 1] = mx;
  }
}

// TMA: lane 0 of warp 0 issues bulk stores of `chunk` bytes from smem; every
// `chunk` it waits for the group issued `lag` groups ago and then fences.
template <int LAG>
__global__ void probe_tma(char* dst, size_t per_cta, int chunk, unsigned long long* lat) {
  extern __shared__ __align__(128) char smem[];
  if (threadIdx.x != 0) return;
  char* base = dst + blockIdx.x * per_cta;
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  unsigned long long sw = 0, sf = 0, mx = 0;
  int cnt = 0;
  for (size_t off = 0; off < per_cta; off += chunk) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(base + off), "r"(s), "r"(chunk)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    unsigned long long t0 = gt();
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(LAG) : "memory");
    unsigned long long t1 = gt();
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    unsigned long long t2 = gt();
    sw += t1 - t0;
    sf += t2 - t1;
    mx = (t2 - t0) > mx ? (t2 - t0) : mx;
    ++cnt;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  lat[blockIdx.x * 3] = sw / cnt;
  lat[blockIdx.x * 3 + 1] = sf / cnt;
  lat[blockIdx.x * 3 + 2] = mx;
}

int main() {
  const size_t bytes = 512ull << 20;
  char *dst, *src;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&dst, bytes));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&src, bytes));
  unsigned long long* lat;
  CK(cudaMallocManaged(&lat, 4096 * 8));
  CK(cudaFuncSetAttribute(probe_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 << 10));
  CK(cudaFuncSetAttribute(probe_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 << 10));
  CK(cudaFuncSetAttribute(probe_tma<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 << 10));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  printf("[\n");
  for (int grid : {32, 128}) {
    for (int pushers : {0, 4, 12}) {
      size_t per = bytes / grid / 16 * 16;
      CK(cudaEventRecord(a));
      probe_stores_v2<<<grid, (pushers + 1) * 32>>>(dst, per, lat, 20);
      CK(cudaEventRecord(b));
      CK(cudaDeviceSynchronize());
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      double s = 0, m = 0;
      for (int i = 0; i < grid; ++i) { s += lat[2 * i]; m = lat[2 * i + 1] > m ? lat[2 * i + 1] : m; }
      printf(" {\"kind\": \"sm_stores\", \"grid\": %d, \"pushers\": %d, \"GBps\": %.0f, \"fence_mean_us\": %.2f, \"fence_max_us\": %.2f},\n",
             grid, pushers, pushers ? bytes / (ms * 1e-3) / 1e9 : 0.0, s / grid / 1e3, m / 1e3);
    }
    for (int chunk : {16 << 10, 64 << 10}) {
      size_t per = bytes / grid / chunk * chunk;
      for (int lag : {0, 2, 4}) {
        CK(cudaEventRecord(a));
        if (lag == 0) probe_tma<0><<<grid, 32, chunk>>>(dst, per, chunk, lat);
        if (lag == 2) probe_tma<2><<<grid, 32, chunk>>>(dst, per, chunk, lat);
        if (lag == 4) probe_tma<4><<<grid, 32, chunk>>>(dst, per, chunk, lat);
        CK(cudaEventRecord(b));
        CK(cudaDeviceSynchronize());
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        double sw = 0, sf = 0, m = 0;
        for (int i = 0; i < grid; ++i) { sw += lat[3 * i]; sf += lat[3 * i + 1]; m = lat[3 * i + 2] > m ? lat[3 * i + 2] : m; }
        printf(" {\"kind\": \"tma\", \"grid\": %d, \"chunk\": %d, \"lag\": %d, \"GBps\": %.0f, \"wait_mean_us\": %.2f, \"fence_mean_us\": %.2f, \"max_us\": %.2f},\n",
               grid, chunk, lag, (double)per * grid / (ms * 1e-3) / 1e9, sw / grid / 1e3, sf / grid / 1e3, m / 1e3);
      }
    }
  }
  printf(" {}\n]\n");
  return 0;
}

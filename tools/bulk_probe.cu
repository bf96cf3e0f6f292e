// Bulk-copy (TMA engine) push to a peer GPU with a BOUNDED number of bulk groups in
// flight, and the cost of publishing completion to the peer.  Tuning probe for the
// ring kernel's data path: does bounding the in-flight bytes keep the
// system-scope fence of the signal path short, and at what bandwidth?
//
// Per CTA: lane 0 of warp 0 (the storer) pushes `per_cta` bytes from one shared-memory
// stage to the peer in `stage`-byte cp.async.bulk stores, one bulk group per stage;
// after each commit it waits until at most D groups are pending (cp.async.bulk.wait_group D)
// and hands every completed "slice" (`slice_stages` stages) to lane 0 of warp 1 (the
// signaller) through shared memory.  The signaller publishes the slice count to a flag in
// the peer's memory: fence_mode 0 = fence.acq_rel.sys + relaxed store, 1 = relaxed store
// only (no fence: throughput reference), 2 = the storer itself fences after completion
// (signaller idle).  Recorded: bandwidth one way and both ways, fence latency mean / max.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bulk_probe tools/bulk_probe.cu
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

template <int D>
__global__ void __launch_bounds__(64) bulk_push(char* dst, size_t per_cta, int stage, int slice_stages,
                                                unsigned long long* flag, unsigned long long* lat, int fence_mode) {
  extern __shared__ __align__(128) char smem[];
  __shared__ int s_done;
  if (threadIdx.x == 0) s_done = 0;
  __syncthreads();
  const int nst = (int)(per_cta / stage);
  const int nslices = nst / slice_stages;
  char* base = dst + blockIdx.x * per_cta;
  if (threadIdx.x == 0) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    int published = 0;
    unsigned long long fsum = 0, fmax = 0;
    for (int i = 0; i < nst; ++i) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(base + (size_t)i * stage),
                   "r"(s), "r"(stage) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group %0;" ::"n"(D) : "memory");
      const int complete = i + 1 - D;  // stages known complete
      const int sl = complete > 0 ? complete / slice_stages : 0;
      if (sl > published) {
        if (fence_mode == 2) {
          const unsigned long long t0 = gt();
          asm volatile("fence.acq_rel.sys;" ::: "memory");
          const unsigned long long d = gt() - t0;
          fsum += d;
          fmax = d > fmax ? d : fmax;
          asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(flag + blockIdx.x), "l"((unsigned long long)sl)
                       : "memory");
        } else {
          asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&s_done)),
                       "r"(sl) : "memory");
        }
        published = sl;
      }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (nslices > published) {
      asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&s_done)),
                   "r"(nslices) : "memory");
    }
    if (fence_mode == 2) {
      lat[blockIdx.x * 3] = fsum;
      lat[blockIdx.x * 3 + 1] = fmax;
      lat[blockIdx.x * 3 + 2] = nslices;
    }
  } else if (threadIdx.x == 32 && fence_mode != 2) {
    int published = 0, cnt = 0;
    unsigned long long fsum = 0, fmax = 0;
    while (published < nslices) {
      int d;
      do {
        asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(d) : "r"((unsigned)__cvta_generic_to_shared(&s_done))
                     : "memory");
      } while (d == published);
      const unsigned long long t0 = gt();
      if (fence_mode == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
      const unsigned long long dt = gt() - t0;
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(flag + blockIdx.x), "l"((unsigned long long)d)
                   : "memory");
      fsum += dt;
      fmax = dt > fmax ? dt : fmax;
      ++cnt;
      published = d;
    }
    lat[blockIdx.x * 3] = fsum;
    lat[blockIdx.x * 3 + 1] = fmax;
    lat[blockIdx.x * 3 + 2] = cnt;
  }
}

typedef void (*KFn)(char*, size_t, int, int, unsigned long long*, unsigned long long*, int);

static KFn kern(int d) {
  switch (d) {
    case 0: return bulk_push<0>;
    case 1: return bulk_push<1>;
    case 2: return bulk_push<2>;
    case 3: return bulk_push<3>;
    case 4: return bulk_push<4>;
    default: return bulk_push<8>;
  }
}

int main(int argc, char** argv) {
  const size_t bytes = 256ull << 20;
  char* dst[2];
  unsigned long long* flag[2];
  unsigned long long* lat[2];
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceEnablePeerAccess(1 - g, 0));
    CK(cudaMalloc(&dst[g], bytes + (64 << 20)));
    CK(cudaMalloc(&flag[g], 4096 * 8));
    CK(cudaMallocManaged(&lat[g], 4096 * 3 * 8));
    for (int d : {0, 1, 2, 3, 4, 8}) CK(cudaFuncSetAttribute(kern(d), cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10));
  }
  cudaStream_t st[2];
  cudaEvent_t ea[2], eb[2];
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaStreamCreate(&st[g]));
    CK(cudaEventCreate(&ea[g]));
    CK(cudaEventCreate(&eb[g]));
  }
  printf("[\n");
  bool first = true;
  for (int grid : {148, 296}) {
    for (int stage : {8 << 10, 16 << 10, 32 << 10, 64 << 10}) {
      for (int D : {0, 1, 2, 4, 8}) {
        for (int fm : {0, 1, 2}) {
          for (int both : {0, 1}) {
            const size_t per = bytes / grid / (4 * stage) * (4 * stage);
            float ms[2] = {0, 0};
            for (int rep = 0; rep < 2; ++rep) {  // rep 0: warm-up
              for (int g = 0; g < (both ? 2 : 1); ++g) {
                CK(cudaSetDevice(g));
                CK(cudaEventRecord(ea[g], st[g]));
                kern(D)<<<grid, 64, stage, st[g]>>>(dst[1 - g], per, stage, 4, flag[1 - g], lat[g], fm);
                CK(cudaGetLastError());
                CK(cudaEventRecord(eb[g], st[g]));
              }
              for (int g = 0; g < (both ? 2 : 1); ++g) {
                CK(cudaSetDevice(g));
                CK(cudaStreamSynchronize(st[g]));
                CK(cudaEventElapsedTime(&ms[g], ea[g], eb[g]));
              }
            }
            double fs = 0, fx = 0, n = 0;
            for (int i = 0; i < grid; ++i) {
              fs += lat[0][3 * i];
              fx = lat[0][3 * i + 1] > fx ? lat[0][3 * i + 1] : fx;
              n += lat[0][3 * i + 2];
            }
            const double t = both ? (ms[0] > ms[1] ? ms[0] : ms[1]) : ms[0];
            printf("%s {\"grid\": %d, \"stage\": %d, \"D\": %d, \"fence_mode\": %d, \"both\": %d, "
                   "\"inflight_MB\": %.2f, \"GBps_per_dir\": %.1f, \"fence_mean_us\": %.2f, \"fence_max_us\": %.2f}\n",
                   first ? " " : ",", grid, stage, D, fm, both, (double)grid * (D + 1) * stage / 1e6,
                   (double)per * grid / (t * 1e-3) / 1e9, n ? fs / n / 1e3 : 0.0, fx / 1e3);
            first = false;
            fflush(stdout);
          }
        }
      }
    }
  }
  printf("]\n");
  return 0;
}

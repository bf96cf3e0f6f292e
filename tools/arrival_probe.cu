// When does pushed data ARRIVE at the peer, compared with the flag that publishes it?
// Tuning / safety probe for the ring kernel's signal path.
//
// Both GPUs run the same kernel at once (both NVLink directions loaded).  CTA b:
//   warp 0 (storer)    pushes nst stages of `stage` bytes from shared memory to the peer
//                      (cp.async.bulk, one group per stage, cp.async.bulk.wait_group D after
//                      each commit); the last 16 B of stage i carry the stamp i+1; every
//                      `slice` completed stages are handed to warp 1 through shared memory
//   warp 1 (signaller) publishes the completed slice count in the peer's flag word:
//                      fence_mode 0 = fence.acq_rel.sys then a relaxed store, 1 = relaxed
//                      store only (no fence)
//   warp 2 (data rx)   polls the stamps the PEER's CTA b writes into this GPU, records the
//                      %globaltimer time each stage's stamp appears
//   warp 3 (flag rx)   polls the flag the peer's CTA b writes here, records when each
//                      slice count appears
// Both receive times are on this GPU's clock: flag - data of a slice's last stage is what
// the publish costs beyond the data's own arrival.  A flag seen BEFORE its slice's last
// stamp (fence_mode 1) would show that bulk-group completion does not order later stores.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/arrival_probe tools/arrival_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

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
__device__ __forceinline__ unsigned long long ld_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

constexpr int kBufs = 4;

template <int D>
__global__ void __launch_bounds__(128) arrival(char* peer, const char* mine, size_t per_cta, int stage, int slice,
                                               unsigned long long* peer_flag, const unsigned long long* my_flag,
                                               unsigned long long epoch, unsigned long long* t_data,
                                               unsigned long long* t_flag, int fence_mode,
                                               unsigned long long* stale) {
  extern __shared__ __align__(128) char smem[];
  __shared__ int s_done;
  if (threadIdx.x == 0) s_done = 0;
  __syncthreads();
  const int nst = (int)(per_cta / stage);
  const int nsl = nst / slice;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane != 0) return;
  if (warp == 0) {
    char* base = peer + blockIdx.x * per_cta;
    int published = 0;
    for (int i = 0; i < nst; ++i) {
      char* sb = smem + (i % kBufs) * stage;
      unsigned long long* st = reinterpret_cast<unsigned long long*>(sb + stage - 16);
      st[0] = epoch * 1000000ull + i + 1;
      st[1] = 0;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(base + (size_t)i * stage),
                   "r"((unsigned)__cvta_generic_to_shared(sb)), "r"(stage) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group %0;" ::"n"(D) : "memory");
      const int complete = i + 1 - D;
      const int sl = complete > 0 ? complete / slice : 0;
      if (sl > published) {
        asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&s_done)), "r"(sl)
                     : "memory");
        published = sl;
      }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&s_done)), "r"(nsl)
                 : "memory");
  } else if (warp == 1) {
    int published = 0;
    while (published < nsl) {
      int d;
      do {
        asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(d) : "r"((unsigned)__cvta_generic_to_shared(&s_done))
                     : "memory");
      } while (d == published);
      if (fence_mode == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(peer_flag + blockIdx.x),
                   "l"(epoch * 1000000ull + (unsigned long long)d) : "memory");
      published = d;
    }
  } else if (warp == 2) {
    const char* base = mine + blockIdx.x * per_cta;
    for (int i = 0; i < nst; ++i) {
      const unsigned long long* st = reinterpret_cast<const unsigned long long*>(base + (size_t)i * stage + stage - 16);
      const unsigned long long want = epoch * 1000000ull + i + 1;
      unsigned long long t0 = gt();
      while (ld_sys(st) != want) {
        if (gt() - t0 > 2000000000ull) break;  // 2 s: give up (recorded as 0)
      }
      t_data[(size_t)blockIdx.x * nst + i] = ld_sys(st) == want ? gt() : 0;
    }
  } else {
    for (int s = 0; s < nsl; ++s) {
      const unsigned long long want = epoch * 1000000ull + s + 1;
      unsigned long long t0 = gt();
      while (ld_sys(my_flag + blockIdx.x) < want) {
        if (gt() - t0 > 2000000000ull) break;
      }
      // acquire the flag, then read back the stamps of every stage of slices <= s: a
      // stale one means the publish did not make the data visible (memory-model test)
      unsigned long long f;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(f) : "l"(my_flag + blockIdx.x) : "memory");
      t_flag[(size_t)blockIdx.x * nsl + s] = f >= want ? gt() : 0;
      if (f >= want) {
        const char* base = mine + blockIdx.x * per_cta;
        for (int i = s * slice; i < (s + 1) * slice; ++i) {
          const unsigned long long* st =
              reinterpret_cast<const unsigned long long*>(base + (size_t)i * stage + stage - 16);
          if (ld_sys(st) != epoch * 1000000ull + i + 1) atomicAdd(stale, 1ull);
        }
      }
    }
  }
}

typedef void (*KFn)(char*, const char*, size_t, int, int, unsigned long long*, const unsigned long long*,
                    unsigned long long, unsigned long long*, unsigned long long*, int, unsigned long long*);
static KFn kern(int d) {
  switch (d) {
    case 0: return arrival<0>;
    case 1: return arrival<1>;
    default: return arrival<2>;
  }
}

int main() {
  const size_t bytes = 128ull << 20;
  char* buf[2];
  unsigned long long *flag[2], *td[2], *tf[2], *stale[2];
  cudaStream_t st[2];
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceEnablePeerAccess(1 - g, 0));
    CK(cudaMalloc(&buf[g], bytes));
    CK(cudaMemset(buf[g], 0, bytes));
    CK(cudaMalloc(&flag[g], 4096 * 8));
    CK(cudaMemset(flag[g], 0, 4096 * 8));
    CK(cudaMalloc(&td[g], (bytes / 4096) * 8));
    CK(cudaMalloc(&tf[g], (bytes / 4096) * 8));
    CK(cudaStreamCreate(&st[g]));
    CK(cudaMallocManaged(&stale[g], 8));
    for (int d = 0; d < 3; ++d)
      CK(cudaFuncSetAttribute(kern(d), cudaFuncAttributeMaxDynamicSharedMemorySize, kBufs * (32 << 10)));
  }
  unsigned long long epoch = 0;
  printf("[\n");
  bool first = true;
  for (int grid : {148}) {
    for (int stage : {8 << 10, 16 << 10, 32 << 10}) {
      for (int D : {0, 1, 2}) {
        for (int fm : {0, 1}) {
          const int slice = (64 << 10) / stage;  // 64 KiB slices
          const size_t per = bytes / grid / (64 << 10) * (64 << 10);
          const int nst = (int)(per / stage), nsl = nst / slice;
          ++epoch;
          *stale[0] = *stale[1] = 0;
          cudaEvent_t a[2], b[2];
          for (int g = 0; g < 2; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaEventCreate(&a[g]));
            CK(cudaEventCreate(&b[g]));
            CK(cudaEventRecord(a[g], st[g]));
            kern(D)<<<grid, 128, kBufs * stage, st[g]>>>(buf[1 - g], buf[g], per, stage, slice, flag[1 - g], flag[g],
                                                         epoch, td[g], tf[g], fm, stale[g]);
            CK(cudaGetLastError());
            CK(cudaEventRecord(b[g], st[g]));
          }
          float ms = 0;
          std::vector<double> lag;  // flag - last stamp of the slice, us
          long neg = 0, missing = 0;
          for (int g = 0; g < 2; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaStreamSynchronize(st[g]));
            float m;
            CK(cudaEventElapsedTime(&m, a[g], b[g]));
            ms = std::max(ms, m);
            std::vector<unsigned long long> hd((size_t)grid * nst), hf((size_t)grid * nsl);
            CK(cudaMemcpy(hd.data(), td[g], hd.size() * 8, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(hf.data(), tf[g], hf.size() * 8, cudaMemcpyDeviceToHost));
            for (int c = 0; c < grid; ++c)
              for (int s = 0; s < nsl; ++s) {
                const unsigned long long f = hf[(size_t)c * nsl + s];
                unsigned long long dmax = 0;
                bool miss = !f;
                for (int i = s * slice; i < (s + 1) * slice; ++i) {
                  const unsigned long long x = hd[(size_t)c * nst + i];
                  miss = miss || !x;
                  dmax = std::max(dmax, x);
                }
                if (miss) { ++missing; continue; }
                const double l = ((double)f - (double)dmax) / 1e3;
                if (l < 0) ++neg;
                lag.push_back(l);
              }
          }
          std::sort(lag.begin(), lag.end());
          auto pct = [&](double p) { return lag.empty() ? 0.0 : lag[(size_t)(p * (lag.size() - 1))]; };
          printf("%s {\"grid\": %d, \"stage\": %d, \"D\": %d, \"fence_mode\": %d, \"GBps_per_dir\": %.1f, "
                 "\"flag_minus_data_us\": {\"p10\": %.2f, \"p50\": %.2f, \"p90\": %.2f, \"max\": %.2f, \"min\": %.2f}, "
                 "\"flag_before_data\": %ld, \"slices\": %zu, \"missing\": %ld, \"stale_after_acquire\": %llu}\n",
                 first ? " " : ",", grid, stage, D, fm, (double)per * grid / (ms * 1e-3) / 1e9, pct(0.1), pct(0.5),
                 pct(0.9), lag.empty() ? 0.0 : lag.back(), lag.empty() ? 0.0 : lag.front(), neg, lag.size(), missing,
                 *stale[0] + *stale[1]);
          first = false;
          fflush(stdout);
        }
      }
    }
  }
  printf("]\n");
  return 0;
}

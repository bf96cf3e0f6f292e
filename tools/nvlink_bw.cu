// NVLink 5 bandwidth probe between GPU 0 and GPU 1 (one process, P2P enabled).
// Measures what the ring kernel's data movement can reach: SM stores (16/32 B),
// SM loads from the peer (pull), TMA bulk stores smem -> peer, and the copy
// engines, one direction and both directions at once.  Tuning tool only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvlink_bw tools/nvlink_bw.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

struct V32 { uint32_t w[8]; };

__global__ void push_v8(const char* __restrict__ src, char* __restrict__ dst, size_t bytes) {
  size_t n = bytes / 32;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    V32 v;
    asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]), "=r"(v.w[5]),
                   "=r"(v.w[6]), "=r"(v.w[7])
                 : "l"(src + i * 32));
    asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + i * 32), "r"(v.w[0]),
                 "r"(v.w[1]), "r"(v.w[2]), "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]), "r"(v.w[7])
                 : "memory");
  }
}

__global__ void push_v4(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t bytes) {
  size_t n = bytes / 16;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = __ldcg(src + i);
}

// store-only (no local read): isolates the NVLink write path
__global__ void store_only_v8(char* __restrict__ dst, size_t bytes) {
  size_t n = bytes / 32;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i;
    asm volatile("st.global.v8.u32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(dst + i * 32), "r"(x) : "memory");
  }
}

// pull: load from the peer, store locally
__global__ void pull_v4(const uint4* __restrict__ peer, uint4* __restrict__ dst, size_t bytes) {
  size_t n = bytes / 16;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = __ldcg(peer + i);
}

// TMA bulk store: each CTA copies its contiguous share from a smem staging buffer
// (content irrelevant) to the peer in `chunk`-byte bulk copies, `depth` in flight.
__global__ void tma_push(char* __restrict__ dst, size_t bytes, int chunk, int depth) {
  extern __shared__ __align__(128) char smem[];
  size_t per = (bytes / gridDim.x) / chunk * chunk;
  char* base = dst + blockIdx.x * per;
  if (threadIdx.x == 0) {
    uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    int inflight = 0;
    for (size_t off = 0; off < per; off += chunk) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(base + off), "r"(s),
                   "r"(chunk)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (++inflight >= depth) {
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(0) : "memory");
        inflight = 0;
      }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// TMA bulk pull: one thread per CTA streams its share of the PEER buffer into a
// ring of `depth` shared-memory stages (mbarrier transaction counts, no fences).
__global__ void tma_pull(const char* __restrict__ src, size_t bytes, int chunk, int depth) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) unsigned long long bars[16];
  if (threadIdx.x != 0) return;
  const size_t per = (bytes / gridDim.x) / chunk * chunk;
  const char* base = src + blockIdx.x * per;
  for (int i = 0; i < depth; ++i) {
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[i]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t n = per / chunk;
  uint32_t phase[16] = {0};
  for (size_t i = 0; i < n + depth; ++i) {
    if (i >= (size_t)depth) {  // retire the load issued depth iterations ago
      const int st = (i - depth) % depth;
      uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[st]);
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(b), "r"(phase[st]) : "memory");
      phase[st] ^= 1;
    }
    if (i < n) {
      const int st = i % depth;
      uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[st]);
      uint32_t d = (uint32_t)__cvta_generic_to_shared(smem + (size_t)st * chunk);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(d), "l"(base + i * chunk), "r"(chunk), "r"(b) : "memory");
    }
  }
}

struct Res { double uni, bi; };

template <class F>
Res measure(F launch, size_t bytes, int iters, char** dsts, char** srcs, cudaStream_t* st) {
  cudaEvent_t a[2], b[2];
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaEventCreate(&a[g]));
    CK(cudaEventCreate(&b[g]));
  }
  Res r;
  // unidirectional: GPU0 -> GPU1
  CK(cudaSetDevice(0));
  for (int i = 0; i < 2; ++i) launch(0, st[0], dsts[1], srcs[0]);
  CK(cudaEventRecord(a[0], st[0]));
  for (int i = 0; i < iters; ++i) launch(0, st[0], dsts[1], srcs[0]);
  CK(cudaEventRecord(b[0], st[0]));
  CK(cudaEventSynchronize(b[0]));
  float ms;
  CK(cudaEventElapsedTime(&ms, a[0], b[0]));
  r.uni = bytes * (double)iters / (ms * 1e-3) / 1e9;
  // bidirectional: both at once
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceSynchronize());
  }
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaEventRecord(a[g], st[g]));
    for (int i = 0; i < iters; ++i) launch(g, st[g], dsts[1 - g], srcs[g]);
    CK(cudaEventRecord(b[g], st[g]));
  }
  double worst = 0;
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaEventSynchronize(b[g]));
    CK(cudaEventElapsedTime(&ms, a[g], b[g]));
    if (ms > worst) worst = ms;
  }
  r.bi = bytes * (double)iters / (worst * 1e-3) / 1e9;
  return r;
}

int main(int argc, char** argv) {
  size_t bytes = (argc > 1 ? atoll(argv[1]) : 256) << 20;
  int iters = 10;
  char* bufs[2];
  char* srcs[2];
  cudaStream_t st[2];
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceEnablePeerAccess(1 - g, 0));
    CK(cudaMalloc(&bufs[g], bytes));
    CK(cudaMalloc(&srcs[g], bytes));
    CK(cudaMemset(srcs[g], 1, bytes));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaFuncSetAttribute(tma_push, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10));
    CK(cudaFuncSetAttribute(tma_pull, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10));
  }
  printf("{\"bytes\": %zu, \"results\": [\n", bytes);
  bool first = true;
  auto out = [&](const char* name, int grid, int thr, Res r) {
    printf("%s {\"kind\": \"%s\", \"grid\": %d, \"threads\": %d, \"uni_GBps\": %.1f, \"bi_GBps_per_dir\": %.1f}\n",
           first ? "" : ",", name, grid, thr, r.uni, r.bi);
    first = false;
    fflush(stdout);
  };
  const bool pull_only = argc > 2 && !strcmp(argv[2], "pull");
  int grids[] = {16, 32, 64, 132, 148, 296};
  for (int gi = 0; gi < 6; ++gi) {
    int grid = grids[gi];
    for (int chunk : {16 << 10, 32 << 10, 64 << 10}) {
      for (int depth : {2, 3, 4, 6}) {
        if ((size_t)chunk * depth > (200u << 10)) continue;
        char nm[64];
        snprintf(nm, sizeof nm, "tma_pull_%dK_d%d", chunk >> 10, depth);
        out(nm, grid, 32, measure([&](int g, cudaStream_t s, char*, char*) {
              tma_pull<<<grid, 32, (size_t)chunk * depth, s>>>(srcs[1 - g], bytes, chunk, depth); }, bytes, iters, bufs,
              srcs, st));
      }
    }
  }
  for (int gi = 0; gi < 6 && !pull_only; ++gi) {
    int grid = grids[gi];
    for (int thr : {256, 512, 1024}) {
      out("push_v8", grid, thr, measure([&](int, cudaStream_t s, char* d, char* src) {
            push_v8<<<grid, thr, 0, s>>>(src, d, bytes); }, bytes, iters, bufs, srcs, st));
      out("push_v4", grid, thr, measure([&](int, cudaStream_t s, char* d, char* src) {
            push_v4<<<grid, thr, 0, s>>>((const uint4*)src, (uint4*)d, bytes); }, bytes, iters, bufs, srcs, st));
      out("store_only_v8", grid, thr, measure([&](int, cudaStream_t s, char* d, char*) {
            store_only_v8<<<grid, thr, 0, s>>>(d, bytes); }, bytes, iters, bufs, srcs, st));
      // pull: GPU g reads from the other GPU's src into its own buf
      out("pull_v4", grid, thr, measure([&](int g, cudaStream_t s, char* d, char*) {
            pull_v4<<<grid, thr, 0, s>>>((const uint4*)srcs[1 - g], (uint4*)bufs[g], bytes); }, bytes, iters, bufs,
            srcs, st));
    }
    for (int chunk : {16 << 10, 64 << 10}) {
      for (int depth : {2, 4, 8}) {
        char nm[64];
        snprintf(nm, sizeof nm, "tma_push_%dK_d%d", chunk >> 10, depth);
        out(nm, grid, 32, measure([&](int, cudaStream_t s, char* d, char*) {
              tma_push<<<grid, 32, chunk, s>>>(d, bytes, chunk, depth); }, bytes, iters, bufs, srcs, st));
      }
    }
  }
  out("memcpy_peer", 0, 0, measure([&](int g, cudaStream_t s, char* d, char* src) {
        CK(cudaMemcpyPeerAsync(d, 1 - g, src, g, bytes, s)); }, bytes, iters, bufs, srcs, st));
  printf("]}\n");
  return 0;
}

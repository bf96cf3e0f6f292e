// Does a GPU push more bytes per second to two peers than to one?  SM-store push
// (st.global.v8, 32 B per thread) from GPU 0 into peer memory: all CTAs to GPU 1, or half
// to GPU 1 and half to GPU 2 (what a bidirectional ring would do).  Also the symmetric
// case where GPUs 1 and 2 push back at the same time.  One process, peer access.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/egress_probe tools/egress_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) {                                                            \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);   \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

// CTAs [0, split) write dst_a, the rest dst_b; each CTA a contiguous share.
__global__ void push2(char* dst_a, char* dst_b, size_t bytes_each, int split) {
  const int cta = blockIdx.x;
  const bool a = cta < split;
  const int idx = a ? cta : cta - split;
  const int n = a ? split : gridDim.x - split;
  char* dst = a ? dst_a : dst_b;
  const size_t per = bytes_each / n / 32 * 32;
  char* p = dst + (size_t)idx * per;
  const unsigned x = 0x3f800000u + cta;
  for (size_t i = threadIdx.x * 32; i < per; i += blockDim.x * 32)
    asm volatile("st.global.v8.u32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p + i), "r"(x) : "memory");
}

int main() {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 3) {
    printf("{\"error\": \"needs 3 GPUs\"}\n");
    return 0;
  }
  const size_t bytes = 256ull << 20;
  char* buf[3];
  for (int d = 0; d < 3; ++d) {
    CK(cudaSetDevice(d));
    for (int e = 0; e < 3; ++e)
      if (e != d) {
        cudaError_t r = cudaDeviceEnablePeerAccess(e, 0);
        if (r != cudaSuccess && r != cudaErrorPeerAccessAlreadyEnabled) CK(r);
        cudaGetLastError();
      }
    CK(cudaMalloc(&buf[d], 2 * bytes));
  }
  auto run = [&](int grid, int threads, bool two, bool both) -> double {
    cudaEvent_t e0, e1;
    CK(cudaSetDevice(0));
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
      for (int d = 0; d < 3; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceSynchronize());
      }
      CK(cudaSetDevice(0));
      CK(cudaEventRecord(e0));
      // GPU 0 pushes `bytes` in total: to GPU 1 only, or half to GPU 1 and half to GPU 2
      if (two) push2<<<grid, threads>>>(buf[1], buf[2] + bytes, bytes / 2, grid / 2);
      else push2<<<grid, threads>>>(buf[1], buf[1] + bytes / 2, bytes / 2, grid / 2);
      CK(cudaEventRecord(e1));
      if (both) {  // the peers push back at the same time (GPU 1 -> 0 [and 2], GPU 2 -> 0 [and 1])
        CK(cudaSetDevice(1));
        if (two) push2<<<grid, threads>>>(buf[0], buf[2], bytes / 2, grid / 2);
        else push2<<<grid, threads>>>(buf[0], buf[0] + bytes / 2, bytes / 2, grid / 2);
        CK(cudaSetDevice(2));
        if (two) push2<<<grid, threads>>>(buf[0] + bytes, buf[1] + bytes, bytes / 2, grid / 2);
        else push2<<<grid, threads>>>(buf[1] + bytes, buf[1] + bytes + bytes / 2, bytes / 2, grid / 2);
      }
      CK(cudaSetDevice(0));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) best = ms;
    }
    for (int d = 0; d < 3; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaDeviceSynchronize());
    }
    return bytes / (best * 1e-3) / 1e9;
  };
  printf("[\n");
  bool first = true;
  for (int grid : {64, 148, 296})
    for (int threads : {256, 512})
      for (int both = 0; both < 2; ++both) {
        const double one = run(grid, threads, false, both);
        const double two = run(grid, threads, true, both);
        printf("%s{\"grid\": %d, \"threads\": %d, \"peers_push_back\": %d, \"one_peer_GBps\": %.1f, "
               "\"two_peers_GBps\": %.1f}",
               first ? "" : ",\n", grid, threads, both, one, two);
        first = false;
      }
  printf("\n]\n");
  return 0;
}

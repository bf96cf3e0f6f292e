// Does NVLink deliver one warp store of a 128-byte line whole?  (Evidence for a
// possible flag-in-line protocol.)  GPU 0 streams lines into
// GPU 1's memory: 8 lanes of a warp each store 16 B with one st.v2.u64, every
// 8-byte word of line i carries the same sequence number and the last word is
// the flag.  GPU 1 (running at the same time) polls each line's flag word, then
// reads the whole line and counts lines whose words disagree ("torn").  PTX does
// not promise 128-byte single-copy atomicity, so a zero count is evidence, not
// proof.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ll128_probe tools/ll128_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
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

// one warp per group of lines; lanes 0..7 store the 8 x 16 B of a line, lanes 8..31
// the next three lines (a warp store covers 4 lines = 512 B, as in NCCL's LL128)
__global__ void sender(unsigned long long* dst, unsigned long long nlines, unsigned long long seq) {
  const unsigned long long warp = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) / 32;
  const unsigned long long nwarps = (gridDim.x * (unsigned long long)blockDim.x) / 32;
  const int lane = threadIdx.x % 32;
  for (unsigned long long g = warp; g * 4 < nlines; g += nwarps) {
    const unsigned long long line = g * 4 + lane / 8;
    if (line >= nlines) continue;
    unsigned long long* p = dst + line * 16 + (lane % 8) * 2;
    const unsigned long long v = (seq << 32) | (line & 0xffffffffull);
    asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1,%2};" ::"l"(p), "l"(v), "l"(v) : "memory");
  }
}

__global__ void receiver(const unsigned long long* buf, unsigned long long nlines, unsigned long long seq,
                         unsigned long long* torn, unsigned long long* checked) {
  const unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  const unsigned long long nt = gridDim.x * (unsigned long long)blockDim.x;
  unsigned long long my_torn = 0, my_checked = 0;
  for (unsigned long long line = t; line < nlines; line += nt) {
    const unsigned long long want = (seq << 32) | (line & 0xffffffffull);
    const unsigned long long* p = buf + line * 16;
    unsigned long long f;
    unsigned spins = 0;
    do {
      asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(f) : "l"(p + 15) : "memory");
      if (++spins > (1u << 26)) break;  // give up on a line (reported as torn)
    } while (f != want);
    bool ok = f == want;
    for (int w = 0; w < 15 && ok; w += 2) {
      unsigned long long a, b;
      asm volatile("ld.relaxed.sys.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p + w) : "memory");
      ok = a == want && (w + 1 == 15 || b == want);
    }
    my_torn += ok ? 0 : 1;
    ++my_checked;
  }
  atomicAdd(torn, my_torn);
  atomicAdd(checked, my_checked);
}

int main(int argc, char** argv) {
  const int passes = argc > 1 ? atoi(argv[1]) : 8;
  const size_t bytes = 1ull << 30;
  const unsigned long long nlines = bytes / 128;
  unsigned long long *buf, *cnt;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMallocManaged(&cnt, 2 * sizeof(unsigned long long)));
  CK(cudaMemset(buf, 0, bytes));
  CK(cudaDeviceSynchronize());
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  cudaStream_t s0, s1;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CK(cudaSetDevice(1));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  unsigned long long total_torn = 0, total_checked = 0;
  for (int pass = 1; pass <= passes; ++pass) {
    cnt[0] = cnt[1] = 0;
    CK(cudaSetDevice(1));
    receiver<<<148 * 4, 256, 0, s1>>>(buf, nlines, (unsigned long long)pass, cnt, cnt + 1);  // polls first
    CK(cudaSetDevice(0));
    sender<<<148 * 2, 512, 0, s0>>>(buf, nlines, (unsigned long long)pass);
    CK(cudaStreamSynchronize(s0));
    CK(cudaSetDevice(1));
    CK(cudaStreamSynchronize(s1));
    total_torn += cnt[0];
    total_checked += cnt[1];
  }
  printf("{\"lines_checked\": %llu, \"torn_lines\": %llu, \"passes\": %d, \"line_bytes\": 128}\n", total_checked,
         total_torn, passes);
  return 0;
}

// sm_100a kernels of the fused ring allreduce (Horovod, arXiv 1802.05799).
//
//   pack    Tensor Fusion step 3 fused with the averaging scale (R1)
//   ring    the 2(N-1) ring iterations pushing into the successor's HBM
//           over NVLink 5 / NVSwitch, with per-channel acquire/release signal counters
//   unpack  Tensor Fusion step 5
//
// Bit-exactness with the oracle relies on: no FMA contraction (-fmad=false and
// explicit __fmul_rn/__fadd_rn), round-to-nearest-even bf16 casts, and the ring
// reduction order of chunk c being the left fold x_c, x_{c+1}, ..., x_{c+N-1}.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "hvd_internal.h"

namespace hvd {
namespace {

constexpr int kHvdErrTimeout = -5;  // HVD_ERR_TIMEOUT

// ------------------------------------------------------------------ memory helpers
struct V32 { uint32_t w[8]; };

// Local data that a peer may have written during this launch: read at L2 (.cg),
// never from a possibly stale L1 line.
__device__ __forceinline__ V32 ld_cg_v8(const void* p) {
  V32 r;
  asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]),
                 "=r"(r.w[5]), "=r"(r.w[6]), "=r"(r.w[7])
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_v8(void* p, const V32& v) {
  asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]),
               "r"(v.w[1]), "r"(v.w[2]), "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]),
               "r"(v.w[7])
               : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ------------------------------------------------------------------ element ops
// Each op works on 32-bit words of a vector (the wire layout) and on single
// elements (ragged tails).  R4: bf16 adds go through fp32 and round RNE.
__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);  // cvt.rn.bf16x2.f32
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ uint16_t f32_to_bf16_bits(float x) {
  __nv_bfloat16 h = __float2bfloat16_rn(x);
  return *reinterpret_cast<uint16_t*>(&h);
}

struct OpF32 {
  using E = float;
  static constexpr int kEsz = 4;
  __device__ static __forceinline__ void add_words(V32& a, const V32& b) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a.w[i] = __float_as_uint(__fadd_rn(__uint_as_float(a.w[i]), __uint_as_float(b.w[i])));
  }
  __device__ static __forceinline__ E add(E a, E b) { return __fadd_rn(a, b); }
};

struct OpBF16 {
  using E = uint16_t;
  static constexpr int kEsz = 2;
  __device__ static __forceinline__ void add_words(V32& a, const V32& b) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      a.w[i] = pack_bf16x2(__fadd_rn(bf16lo(a.w[i]), bf16lo(b.w[i])),
                           __fadd_rn(bf16hi(a.w[i]), bf16hi(b.w[i])));
  }
  __device__ static __forceinline__ E add(E a, E b) {
    return f32_to_bf16_bits(__fadd_rn(__uint_as_float(uint32_t(a) << 16), __uint_as_float(uint32_t(b) << 16)));
  }
};

struct OpI32 {
  using E = uint32_t;  // two's-complement wrap (R11)
  static constexpr int kEsz = 4;
  __device__ static __forceinline__ void add_words(V32& a, const V32& b) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a.w[i] += b.w[i];
  }
  __device__ static __forceinline__ E add(E a, E b) { return a + b; }
};

struct OpI64 {
  using E = unsigned long long;
  static constexpr int kEsz = 8;
  __device__ static __forceinline__ void add_words(V32& a, const V32& b) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      unsigned long long x = (unsigned long long)a.w[2 * i] | ((unsigned long long)a.w[2 * i + 1] << 32);
      unsigned long long y = (unsigned long long)b.w[2 * i] | ((unsigned long long)b.w[2 * i + 1] << 32);
      x += y;
      a.w[2 * i] = uint32_t(x);
      a.w[2 * i + 1] = uint32_t(x >> 32);
    }
  }
  __device__ static __forceinline__ E add(E a, E b) { return a + b; }
};

// ------------------------------------------------------------------ ring kernel
// One slice [lo, hi) of one ring iteration, by one CTA:
//   kCopy:       nbuf/nscratch[lo,hi) <- buf[lo,hi)
//   kAdd:        dst[lo,hi) <- buf[lo,hi) + scratch[lo,hi)       (reduce-scatter)
//   kAddLocal:   buf[lo,hi) and nbuf[lo,hi) <- buf + scratch     (last add, all-gather step 0)
enum SliceKind { kCopy = 0, kAdd = 1, kAddLocal = 2 };

constexpr int kUnroll = 2;  // 2 x (2 x 32 B) loads in flight per thread; 4 spills (wide-register alignment)

template <class Op, int KIND>
__device__ __forceinline__ void do_slice(const char* __restrict__ a, const char* __restrict__ b,
                                         char* __restrict__ dst, char* __restrict__ dst_local,
                                         unsigned long long lo, unsigned long long hi) {
  using E = typename Op::E;
  const unsigned long long nbytes = (hi - lo) * Op::kEsz;
  const unsigned long long nvec = nbytes / 32;
  const char* pa = a + lo * Op::kEsz;
  const char* pb = b + lo * Op::kEsz;
  char* pd = dst + lo * Op::kEsz;
  char* pl = dst_local + lo * Op::kEsz;
  const unsigned nthr = blockDim.x;
  for (unsigned long long v0 = threadIdx.x; v0 < nvec; v0 += (unsigned long long)nthr * kUnroll) {
    V32 x[kUnroll], y[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const unsigned long long v = v0 + (unsigned long long)u * nthr;
      if (v < nvec) {
        x[u] = ld_cg_v8(pa + v * 32);
        if (KIND != kCopy) y[u] = ld_cg_v8(pb + v * 32);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const unsigned long long v = v0 + (unsigned long long)u * nthr;
      if (v < nvec) {
        if (KIND != kCopy) Op::add_words(x[u], y[u]);
        st_v8(pd + v * 32, x[u]);
        if (KIND == kAddLocal) st_v8(pl + v * 32, x[u]);
      }
    }
  }
  // ragged tail (only at the end of the buffer): element by element
  const unsigned long long tail0 = nvec * 32 / Op::kEsz;
  for (unsigned long long e = tail0 + threadIdx.x; e < hi - lo; e += nthr) {
    E x = *reinterpret_cast<const volatile E*>(pa + e * Op::kEsz);
    if (KIND != kCopy) x = Op::add(x, *reinterpret_cast<const volatile E*>(pb + e * Op::kEsz));
    *reinterpret_cast<E*>(pd + e * Op::kEsz) = x;
    if (KIND == kAddLocal) *reinterpret_cast<E*>(pl + e * Op::kEsz) = x;
  }
}

// Thread 0 spins (acquire, system scope) until *flag >= target; the CTA then
// proceeds.  Returns false on watchdog timeout (error latched in host memory).
__device__ __forceinline__ bool wait_signal(const unsigned long long* flag, unsigned long long target,
                                            int* err, unsigned long long timeout_ns) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    int ok = 1;
    if (ld_acquire_sys(flag) < target) {
      const unsigned long long t0 = globaltimer();
      unsigned spins = 0;
      while (ld_acquire_sys(flag) < target) {
        if ((++spins & 1023u) == 0) {
          if (globaltimer() - t0 > timeout_ns || *(volatile int*)err != 0) {
            *(volatile int*)err = kHvdErrTimeout;
            ok = 0;
            break;
          }
        }
      }
    }
    s_ok = ok;
  }
  __syncthreads();
  return s_ok != 0;
}

// All threads make their stores to the successor visible system-wide, then
// thread 0 publishes the counter (release, system scope).
__device__ __forceinline__ void send_signal(unsigned long long* nflag, unsigned long long value) {
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) st_release_sys(nflag, value);
}

__device__ __forceinline__ void slice_range(const RingParams& P, int c, int ch, int k,
                                            unsigned long long& lo, unsigned long long& hi) {
  const unsigned long long L = P.L;
  unsigned long long c_lo = (unsigned long long)c * P.q;
  c_lo = c_lo < L ? c_lo : L;
  unsigned long long c_hi = c_lo + P.q;
  c_hi = c_hi < L ? c_hi : L;
  unsigned long long h_lo = c_lo + (unsigned long long)ch * P.ch_el;
  h_lo = h_lo < c_hi ? h_lo : c_hi;
  unsigned long long h_hi = h_lo + P.ch_el;
  h_hi = h_hi < c_hi ? h_hi : c_hi;
  lo = h_lo + (unsigned long long)k * P.slice_el;
  lo = lo < h_hi ? lo : h_hi;
  hi = lo + P.slice_el;
  hi = hi < h_hi ? hi : h_hi;
}

__device__ __forceinline__ int mod(int a, int n) { return ((a % n) + n) % n; }

// Ring allreduce of one fusion buffer.  grid = (channels, local ranks).
// Iteration t = 0..2N-3 (t < N-1: reduce-scatter step s = t; else all-gather
// step s = t-N+1).  Channel `ch` of rank r owns the ch-th sub-range of every
// chunk and sends one signal per (t, slice k) to the same channel of r+1; it
// waits for the predecessor's signal of (t-1, k) before touching data that
// signal covers.  After the loop it waits for the predecessor's last signal,
// so the kernel completes only when every chunk has arrived.
template <class Op>
__global__ void __launch_bounds__(512, 1) ring_allreduce_kernel(const __grid_constant__ RingParams P) {
  const RingRank& me = P.rk[blockIdx.y];
  const int ch = blockIdx.x;
  const int N = P.N;
  const int r = me.rank;
  const int K = P.K;
  const unsigned long long base = P.base[ch];
  const int T = 2 * (N - 1);
  unsigned long long sent = 0;
  for (int t = 0; t < T; ++t) {
    const bool rs = t < N - 1;
    const int s = rs ? t : t - (N - 1);
    const int c = rs ? mod(r - s, N) : mod(r + 1 - s, N);
    for (int k = 0; k < K; ++k) {
      unsigned long long lo, hi;
      slice_range(P, c, ch, k, lo, hi);
      if (t > 0 && !wait_signal(me.flags + ch, base + (unsigned long long)(t - 1) * K + k + 1, P.err,
                                P.timeout_ns))
        return;
      if (hi > lo) {
        if (rs && s == 0)
          do_slice<Op, kCopy>(me.buf, nullptr, me.nscratch, nullptr, lo, hi);
        else if (rs)
          do_slice<Op, kAdd>(me.buf, me.scratch, me.nscratch, nullptr, lo, hi);
        else if (s == 0)
          do_slice<Op, kAddLocal>(me.buf, me.scratch, me.nbuf, me.buf, lo, hi);
        else
          do_slice<Op, kCopy>(me.buf, nullptr, me.nbuf, nullptr, lo, hi);
        sent += (hi - lo) * Op::kEsz;
      }
      send_signal(me.nflags + ch, base + (unsigned long long)t * K + k + 1);
    }
  }
  if (!wait_signal(me.flags + ch, base + (unsigned long long)T * K, P.err, P.timeout_ns)) return;
  if (threadIdx.x == 0) {
    atomicAdd(me.stats + 0, sent);
    if (ch == 0) atomicAdd(me.stats + 1, (unsigned long long)T);
  }
}

// ------------------------------------------------------------------ pack / unpack
// The fusion buffer is a sequence of 16 B vectors; member s occupies vectors
// [vbeg_s, vbeg_{s+1}).  A tile is `tile_vecs` consecutive vectors; tile_seg
// gives the member of the tile's first and last vector, so each thread finds
// its member by a short binary search inside the tile.
__device__ __forceinline__ int find_seg(const PackParams& P, unsigned long long v, int lo, int hi) {
  while (lo < hi) {  // largest s in [lo, hi] with vbeg[s] <= v
    const int mid = (lo + hi + 1) >> 1;
    if (P.segs[mid].vbeg <= v) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <int ESZ> struct Pack16;

// fp32 -> fp32: x * s with binary32 RN (R1); plain copy when scale is off.
template <> struct Pack16<4> {
  __device__ static __forceinline__ uint4 conv(uint4 x, float s, int on, int dtype) {
    if (on && dtype == 1) {
      x.x = __float_as_uint(__fmul_rn(__uint_as_float(x.x), s));
      x.y = __float_as_uint(__fmul_rn(__uint_as_float(x.y), s));
      x.z = __float_as_uint(__fmul_rn(__uint_as_float(x.z), s));
      x.w = __float_as_uint(__fmul_rn(__uint_as_float(x.w), s));
    }
    return x;
  }
};
template <> struct Pack16<2> {
  __device__ static __forceinline__ uint32_t sc2(uint32_t w, float s) {
    return pack_bf16x2(__fmul_rn(bf16lo(w), s), __fmul_rn(bf16hi(w), s));
  }
  __device__ static __forceinline__ uint4 conv(uint4 x, float s, int on, int) {
    if (on) { x.x = sc2(x.x, s); x.y = sc2(x.y, s); x.z = sc2(x.z, s); x.w = sc2(x.w, s); }
    return x;
  }
};
template <> struct Pack16<8> {
  __device__ static __forceinline__ uint4 conv(uint4 x, float, int, int) { return x; }
};

template <int ESZ>
__device__ __forceinline__ void scale_elem(const char* src, char* dst, float s, int on, int dtype) {
  if (ESZ == 4) {
    uint32_t w = *reinterpret_cast<const uint32_t*>(src);
    if (on && dtype == 1) w = __float_as_uint(__fmul_rn(__uint_as_float(w), s));
    *reinterpret_cast<uint32_t*>(dst) = w;
  } else if (ESZ == 2) {
    uint16_t h = *reinterpret_cast<const uint16_t*>(src);
    if (on) h = f32_to_bf16_bits(__fmul_rn(__uint_as_float(uint32_t(h) << 16), s));
    *reinterpret_cast<uint16_t*>(dst) = h;
  } else {
    *reinterpret_cast<unsigned long long*>(dst) = *reinterpret_cast<const unsigned long long*>(src);
  }
}

template <int ESZ, bool PACK>
__global__ void __launch_bounds__(512) pack_kernel(const __grid_constant__ PackParams P, int dtype) {
  constexpr int VEL = kPackVecBytes / ESZ;
  char* const buf = P.buf[blockIdx.y];
  char* const* src_tab = P.src + (size_t)blockIdx.y * P.nseg;
  for (unsigned long long tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x) {
    const int s_lo = P.tile_seg[tile];
    const int s_hi = P.tile_seg[tile + 1];
    const unsigned long long v0 = tile * P.tile_vecs;
    unsigned long long v1 = v0 + P.tile_vecs;
    v1 = v1 < P.nvec ? v1 : P.nvec;
    int s = s_lo;
    for (unsigned long long v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
      if (s < s_hi && P.segs[s + 1].vbeg <= v) s = find_seg(P, v, s, s_hi);
      const PackSeg sg = P.segs[s];
      const unsigned long long e0 = v * VEL - sg.dst_off;
      char* tens = src_tab[s] + e0 * ESZ;
      char* bvec = buf + v * kPackVecBytes;
      const bool full = e0 + VEL <= sg.count;
      const bool aligned = ((reinterpret_cast<uintptr_t>(tens) & 15) == 0);
      if (PACK) {
        if (full && aligned) {
          uint4 x = __ldcs(reinterpret_cast<const uint4*>(tens));
          *reinterpret_cast<uint4*>(bvec) = Pack16<ESZ>::conv(x, P.scale, P.scale_on, dtype);
        } else {
          alignas(16) char tmp[kPackVecBytes];
#pragma unroll
          for (int i = 0; i < VEL; ++i) {
            if (e0 + i < sg.count) scale_elem<ESZ>(tens + i * ESZ, tmp + i * ESZ, P.scale, P.scale_on, dtype);
            else for (int b = 0; b < ESZ; ++b) tmp[i * ESZ + b] = 0;  // interior padding
          }
          *reinterpret_cast<uint4*>(bvec) = *reinterpret_cast<const uint4*>(tmp);
        }
      } else {
        const uint4 x = __ldcg(reinterpret_cast<const uint4*>(bvec));
        if (full && aligned) {
          __stcs(reinterpret_cast<uint4*>(tens), x);
        } else {
          const char* xb = reinterpret_cast<const char*>(&x);
#pragma unroll
          for (int i = 0; i < VEL; ++i)
            if (e0 + i < sg.count)
              for (int b = 0; b < ESZ; ++b) tens[i * ESZ + b] = xb[i * ESZ + b];
        }
      }
    }
  }
}

struct BufList { char* b[kMaxLocal]; };

template <int ESZ>
__global__ void __launch_bounds__(512) scale_kernel(const BufList bufs, unsigned long long count, float s,
                                                    int dtype) {
  char* buf = bufs.b[blockIdx.y];
  constexpr int VEL = 16 / ESZ;
  const unsigned long long nvec = count / VEL;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long v = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; v < nvec; v += stride) {
    uint4 x = *reinterpret_cast<const uint4*>(buf + v * 16);
    *reinterpret_cast<uint4*>(buf + v * 16) = Pack16<ESZ>::conv(x, s, 1, dtype);
  }
  for (unsigned long long e = nvec * VEL + blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < count;
       e += stride)
    scale_elem<ESZ>(buf + e * ESZ, buf + e * ESZ, s, 1, dtype);
}

}  // namespace

// ------------------------------------------------------------------ launchers
template <bool PACK>
static cudaError_t launch_pack_impl(const PackParams& p, int dtype, int nlocal, int grid, int threads,
                                    cudaStream_t s) {
  if (p.ntiles == 0) return cudaSuccess;
  unsigned long long g = p.ntiles < (unsigned long long)grid ? p.ntiles : (unsigned long long)grid;
  dim3 gd((unsigned)g, nlocal);
  switch (elem_size(dtype)) {
    case 4: pack_kernel<4, PACK><<<gd, threads, 0, s>>>(p, dtype); break;
    case 2: pack_kernel<2, PACK><<<gd, threads, 0, s>>>(p, dtype); break;
    case 8: pack_kernel<8, PACK><<<gd, threads, 0, s>>>(p, dtype); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_pack(const PackParams& p, int dtype, int nlocal, int grid, int threads, cudaStream_t s) {
  return launch_pack_impl<true>(p, dtype, nlocal, grid, threads, s);
}

cudaError_t launch_unpack(const PackParams& p, int dtype, int nlocal, int grid, int threads, cudaStream_t s) {
  return launch_pack_impl<false>(p, dtype, nlocal, grid, threads, s);
}

cudaError_t launch_scale(char* const* bufs, int nlocal, unsigned long long count, int dtype, float scale,
                         int grid, int threads, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  BufList b = {};
  for (int i = 0; i < nlocal && i < kMaxLocal; ++i) b.b[i] = bufs[i];
  dim3 gd(grid, nlocal);
  switch (elem_size(dtype)) {
    case 4: scale_kernel<4><<<gd, threads, 0, s>>>(b, count, scale, dtype); break;
    case 2: scale_kernel<2><<<gd, threads, 0, s>>>(b, count, scale, dtype); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <class Op>
static cudaError_t launch_ring_t(const RingParams& p, int nch, int nlocal, int threads, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nch, nlocal);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (they wait on each other)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, ring_allreduce_kernel<Op>, p);
}

cudaError_t launch_ring(const RingParams& p, int dtype, int nch, int nlocal, int threads, cudaStream_t s) {
  switch (dtype) {
    case 1: return launch_ring_t<OpF32>(p, nch, nlocal, threads, s);
    case 2: return launch_ring_t<OpBF16>(p, nch, nlocal, threads, s);
    case 3: return launch_ring_t<OpI32>(p, nch, nlocal, threads, s);
    case 4: return launch_ring_t<OpI64>(p, nch, nlocal, threads, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t ring_max_ctas_per_sm(int dtype, int threads, int* out) {
  switch (dtype) {
    case 1: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, ring_allreduce_kernel<OpF32>, threads, 0);
    case 2: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, ring_allreduce_kernel<OpBF16>, threads, 0);
    case 3: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, ring_allreduce_kernel<OpI32>, threads, 0);
    case 4: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, ring_allreduce_kernel<OpI64>, threads, 0);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hvd

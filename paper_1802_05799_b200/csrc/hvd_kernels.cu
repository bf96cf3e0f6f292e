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
#include <cstdio>

#include "hvd_internal.h"

namespace hvd {
namespace {

constexpr int kHvdErrTimeout = -5;   // HVD_ERR_TIMEOUT
constexpr int kHvdErrMismatch = -7;  // HVD_ERR_MISMATCH

// The error word kernels see (`err` in RingParams) lives in DEVICE memory: spin loops
// poll it to give up early, and polling host-mapped memory would put a PCIe read in
// every watchdog check — under heavy host<->device copy traffic those reads take so
// long that the polling warps fall behind (measured: LL128 launches of 10 us turned
// into 1.5 ms next to hvd_allreduce_host's copies).  Its second half points to the
// host-mapped word hvd_poll_error reads; raise_err latches the code in both.
struct ErrWords {
  int code;        // device copy (read by spin loops)
  int pad;
  int* host;       // host-mapped word (written on error only)
};
__device__ __forceinline__ void raise_err(int* err, int code) {
  *(volatile int*)err = code;
  int* h = reinterpret_cast<ErrWords*>(err)->host;
  if (h) *(volatile int*)h = code;
  __threadfence_system();
}

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
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ------------------------------------------------------------------ job timeline
// One per kernel, constructed first thing (every thread of the CTA is present, so the
// construction barrier is safe).  Its destructor runs at each thread's return, whichever
// warp-specialised path it took: the last thread of the CTA folds the CTA's end into
// the launch record of its local rank (blockIdx.y), and the last CTA of that rank
// publishes the record to the host-mapped slot and re-arms it (JtRef, hvd_internal.h).
struct JtGuard {
  const JtRef& jt;
  unsigned* left;
  __device__ __forceinline__ explicit JtGuard(const JtRef& j) : jt(j), left(nullptr) {
    if (jt.rec == nullptr) return;
    __shared__ unsigned s_jt_left;
    left = &s_jt_left;
    if (threadIdx.x == 0) {
      s_jt_left = blockDim.x;
      atomicMin(jt.rec + blockIdx.y * kJtWords, globaltimer());
    }
    __syncthreads();
  }
  __device__ __forceinline__ ~JtGuard() {
    if (jt.rec == nullptr) return;
    if (atomicSub(left, 1u) != 1u) return;
    unsigned long long* r = jt.rec + blockIdx.y * kJtWords;
    atomicMax(r + 1, globaltimer());
    __threadfence();
    if (atomicAdd(r + 2, 1ull) != gridDim.x - 1) return;
    __threadfence();
    const unsigned long long b = atomicAdd(r + 0, 0ull), e = atomicAdd(r + 1, 0ull);
    volatile unsigned long long* h = jt.host + blockIdx.y * kJtWords;
    h[1] = b;
    h[2] = e;
    h[3] = gridDim.x;
    __threadfence_system();
    h[0] = jt.seq;
    r[0] = ~0ull;  // re-arm for the launch that reuses this slot (kJtSlots launches later)
    r[1] = 0;
    r[2] = 0;
  }
};

__global__ void jt_clock_kernel(unsigned long long* out) {
  volatile unsigned long long* o = out;
  *o = globaltimer();
  __threadfence_system();
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
  template <int NW>
  __device__ static __forceinline__ void add_words(uint32_t* a, const uint32_t* b) {
#pragma unroll
    for (int i = 0; i < NW; ++i) a[i] = __float_as_uint(__fadd_rn(__uint_as_float(a[i]), __uint_as_float(b[i])));
  }
  __device__ static __forceinline__ E add(E a, E b) { return __fadd_rn(a, b); }
};

struct OpBF16 {
  using E = uint16_t;
  static constexpr int kEsz = 2;
  template <int NW>
  __device__ static __forceinline__ void add_words(uint32_t* a, const uint32_t* b) {
#pragma unroll
    for (int i = 0; i < NW; ++i)
      a[i] = pack_bf16x2(__fadd_rn(bf16lo(a[i]), bf16lo(b[i])), __fadd_rn(bf16hi(a[i]), bf16hi(b[i])));
  }
  __device__ static __forceinline__ E add(E a, E b) {
    return f32_to_bf16_bits(__fadd_rn(__uint_as_float(uint32_t(a) << 16), __uint_as_float(uint32_t(b) << 16)));
  }
};

struct OpI32 {
  using E = uint32_t;  // two's-complement wrap (R11)
  static constexpr int kEsz = 4;
  template <int NW>
  __device__ static __forceinline__ void add_words(uint32_t* a, const uint32_t* b) {
#pragma unroll
    for (int i = 0; i < NW; ++i) a[i] += b[i];
  }
  __device__ static __forceinline__ E add(E a, E b) { return a + b; }
};

struct OpI64 {
  using E = unsigned long long;
  static constexpr int kEsz = 8;
  template <int NW>
  __device__ static __forceinline__ void add_words(uint32_t* a, const uint32_t* b) {
#pragma unroll
    for (int i = 0; i < NW / 2; ++i) {
      unsigned long long x = (unsigned long long)a[2 * i] | ((unsigned long long)a[2 * i + 1] << 32);
      unsigned long long y = (unsigned long long)b[2 * i] | ((unsigned long long)b[2 * i + 1] << 32);
      x += y;
      a[2 * i] = uint32_t(x);
      a[2 * i + 1] = uint32_t(x >> 32);
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

constexpr int kPackBatch = 8;  // == kPackVecsPerThread in the runtime (tile = 256 x 8 vectors)
constexpr int kUnroll = 2;  // 2 x (2 x 32 B) loads in flight per thread (ring_allreduce_kernel: 144 registers, no spills)

template <class Op, int KIND>
__device__ __forceinline__ void do_slice(const char* __restrict__ a, const char* __restrict__ b,
                                         char* __restrict__ dst, char* __restrict__ dst_local,
                                         unsigned long long lo, unsigned long long hi, unsigned tid, unsigned nthr) {
  using E = typename Op::E;
  const unsigned long long nbytes = (hi - lo) * Op::kEsz;
  const unsigned long long nvec = nbytes / 32;
  const char* pa = a + lo * Op::kEsz;
  const char* pb = b + lo * Op::kEsz;
  char* pd = dst + lo * Op::kEsz;
  char* pl = dst_local + lo * Op::kEsz;
  for (unsigned long long v0 = tid; v0 < nvec; v0 += (unsigned long long)nthr * kUnroll) {
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
        if (KIND != kCopy) Op::template add_words<8>(x[u].w, y[u].w);
        st_v8(pd + v * 32, x[u]);
        if (KIND == kAddLocal) st_v8(pl + v * 32, x[u]);
      }
    }
  }
  // ragged tail (only at the end of the buffer): element by element
  const unsigned long long tail0 = nvec * 32 / Op::kEsz;
  for (unsigned long long e = tail0 + tid; e < hi - lo; e += nthr) {
    E x = *reinterpret_cast<const volatile E*>(pa + e * Op::kEsz);
    if (KIND != kCopy) x = Op::add(x, *reinterpret_cast<const volatile E*>(pb + e * Op::kEsz));
    *reinterpret_cast<E*>(pd + e * Op::kEsz) = x;
    if (KIND == kAddLocal) *reinterpret_cast<E*>(pl + e * Op::kEsz) = x;
  }
}

// Named barriers (ids 1..5; 0 is __syncthreads).
__device__ __forceinline__ void bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// The data-warp leader spins (acquire, system scope) until *flag >= target.
// Returns false on watchdog timeout (error latched in host-mapped memory).
__device__ __forceinline__ bool spin_until(const unsigned long long* flag, unsigned long long target, int* err,
                                           unsigned long long timeout_ns) {
  if (ld_acquire_sys(flag) >= target) return true;
  const unsigned long long t0 = globaltimer();
  unsigned spins = 0;
  while (ld_acquire_sys(flag) < target) {
    if ((++spins & 1023u) == 0) {
      if (globaltimer() - t0 > timeout_ns || *(volatile int*)err != 0) {
        raise_err(err, kHvdErrTimeout);
        return false;
      }
    }
  }
  return true;
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

// Ring allreduce of one fusion buffer.  grid = (channels, local ranks);
// block = D data warps + 1 signal warp.
//
// Iteration t = 0..2N-3 (t < N-1: reduce-scatter step s = t; else all-gather
// step s = t-N+1); slice k = 0..K-1; slice sequence number i = t*K + k.
// Channel `ch` of rank r owns the ch-th sub-range of every chunk.
//
// Data warps move slice i (loads at L2, 32 B stores into the successor's HBM).
// Before slice i of iteration t >= 1 their leader waits until the
// predecessor's counter reaches base + (t-1)K + k + 1 (its slice (t-1, k) has
// landed here).  One barrier per slice (data warps only) then both retires
// slice i and releases slice i+1; the leader publishes "i+1 slices done" in
// shared memory (release, CTA scope).
// The signal warp never blocks the data warps: it polls that shared count,
// makes every store of the slices done so far visible system-wide with ONE
// fence.acq_rel.sys (barrier cumulativity covers the data warps' stores) and
// publishes base + done in the successor's counter.  A fence waits for the
// NVLink drain of everything in flight (~us), so one fence covers a batch of
// slices and its latency overlaps the pushes of the next ones.  After the loop
// the leader waits for the predecessor's last counter, so the kernel completes
// only when every chunk has arrived.
constexpr int kBarData = 1;

__device__ __forceinline__ void st_release_cta_shared(int* p, int v) {
  asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_cta_shared64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.cta.shared.u64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_cta_shared64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.cta.shared.u64 %0, [%1];" : "=l"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acquire_cta_shared(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
  return v;
}

// Signal warp body (lane 0): publish progress `*done` to the successor's counter.
__device__ __forceinline__ void signal_loop(const int* done, int total, unsigned long long* nflag,
                                            unsigned long long base, int sig_mode, int* pub = nullptr,
                                            unsigned long long* tl_sig = nullptr, int tl_max = 0) {
  int published = 0, nrec = 0;
  while (published < total) {
    int d;
    while ((d = ld_acquire_cta_shared(done)) == published) __nanosleep(32);
    if (sig_mode == 1) {
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(nflag), "l"(base + (unsigned long long)d) : "memory");
    } else {
      st_release_sys(nflag, base + (unsigned long long)d);
    }
    if (pub) st_release_cta_shared(pub, d);
    if (tl_sig && nrec < tl_max) {
      tl_sig[2 * nrec] = globaltimer();
      tl_sig[2 * nrec + 1] = (unsigned long long)d;
      ++nrec;
    }
    published = d;
  }
}

// Several signal warps (HVD_CFG_SIGNAL_WARPS): a fence under NVLink load takes ~15 us
// (profiles/r02_arrival_probe.json), so one signal lane publishes at most one batch per
// fence.  Here each warp's lane 0 claims the slices done so far, fences and raises the
// successor's counter with a max (publishes may land out of order; the counter stays
// monotone), so fences overlap and a slice waits for at most one fence, not two.
__device__ __forceinline__ void signal_loop_multi(const int* done, int* claimed, int total,
                                                  unsigned long long* nflag, unsigned long long base, int* pub) {
  for (;;) {
    const int c = *(volatile int*)claimed;
    if (c >= total) return;
    const int d = ld_acquire_cta_shared(done);
    if (d <= c) {
      __nanosleep(32);
      continue;
    }
    if (atomicCAS(claimed, c, d) != c) continue;
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    asm volatile("red.relaxed.sys.global.max.u64 [%0], %1;" ::"l"(nflag), "l"(base + (unsigned long long)d) : "memory");
    if (pub) atomicMax(pub, d);
  }
}

template <class Op>
__global__ void __maxnreg__(152) ring_allreduce_kernel(const __grid_constant__ RingParams P) {
  JtGuard jtg(P.jt);
  const RingRank& me = P.rk[blockIdx.y];
  const int ch = blockIdx.x;
  const int N = P.N;
  const int r = me.rank;
  const int K = P.K;
  const unsigned long long base = P.base[ch];
  const int T = 2 * (N - 1);
  const int nd = blockDim.x - 32;  // data threads
  __shared__ int s_abort, s_done;
  if (threadIdx.x == 0) {
    s_abort = 0;
    s_done = 0;
  }
  __syncthreads();

  if (threadIdx.x >= nd) {  // ---- signal warp
    if (threadIdx.x == nd) {
      st_relaxed_sys(me.phash + ch, P.hash);     // handshake: previous launch done with the regions,
      st_release_sys(me.pready + ch, P.epoch);   // and this launch's geometry
      signal_loop(&s_done, T * K, me.nflags + ch, base, P.sig_mode);
    }
    return;
  }

  // ---- data warps
  const unsigned tid = threadIdx.x;
  if (tid == 0) {
    if (!spin_until(me.rflags + ch, P.epoch, P.err, P.timeout_ns)) {
      s_abort = 1;
    } else if (*(volatile const unsigned long long*)(me.rhash + ch) != P.hash) {
      raise_err(P.err, kHvdErrMismatch);
      s_abort = 1;
    }
  }
  bar_sync(kBarData, nd);  // no push before the successor's handshake
  unsigned long long sent = 0;
  int i = 0;
  for (int t = 0; t < T; ++t) {
    const bool rs = t < N - 1;
    const int s = rs ? t : t - (N - 1);
    const int c = rs ? mod(r - s, N) : mod(r + 1 - s, N);
    for (int k = 0; k < K; ++k, ++i) {
      unsigned long long lo, hi;
      slice_range(P, c, ch, k, lo, hi);
      if (hi > lo && !s_abort) {
        if (rs && s == 0)
          do_slice<Op, kCopy>(me.buf, nullptr, me.nscratch, nullptr, lo, hi, tid, nd);
        else if (rs)
          do_slice<Op, kAdd>(me.buf, me.scratch, me.nscratch, nullptr, lo, hi, tid, nd);
        else if (s == 0)
          do_slice<Op, kAddLocal>(me.buf, me.scratch, me.nbuf, me.buf, lo, hi, tid, nd);
        else
          do_slice<Op, kCopy>(me.buf, nullptr, me.nbuf, nullptr, lo, hi, tid, nd);
        sent += (hi - lo) * Op::kEsz;
      }
      // retire slice i (all data warps' stores issued), publish it to the signal
      // warp, THEN wait for the next slice's dependency: publishing first keeps the
      // ring free of cycles (slice i never waits on anything downstream of itself)
      bar_sync(kBarData, nd);
      if (tid == 0) {
        st_release_cta_shared(&s_done, i + 1);
        const int tn = (k + 1 < K) ? t : t + 1;
        const int kn = (k + 1 < K) ? k + 1 : 0;
        // next slice needs the predecessor's (tn-1, kn); after the last slice: its (T-1, K-1)
        unsigned long long target = 0;
        if (tn < T && tn > 0) target = base + (unsigned long long)(tn - 1) * K + kn + 1;
        else if (tn >= T) target = base + (unsigned long long)T * K;
        if (target && !s_abort && !spin_until(me.flags + ch, target, P.err, P.timeout_ns)) s_abort = 1;
      }
      if (t + (k + 1 == K) > 0) bar_sync(kBarData, nd);  // release the next slice (no wait inside step 0)
    }
  }
  if (tid == 0) {
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

// Each thread owns kPackBatch vectors of a tile (stride blockDim) and issues all
// their loads before any store, so kPackBatch x 16 B per thread are in flight.
template <int ESZ, bool PACK>
__global__ void __launch_bounds__(256) pack_kernel(const __grid_constant__ PackParams P, int dtype) {
  JtGuard jtg(P.jt);
  constexpr int VEL = kPackVecBytes / ESZ;
  char* const buf = P.buf[blockIdx.y];
  char* const* src_tab = P.src + (size_t)blockIdx.y * P.nseg;
  for (unsigned long long tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x) {
    const int s_hi = P.tile_seg[tile + 1];
    const unsigned long long v0 = tile * P.tile_vecs;
    unsigned long long v1 = v0 + P.tile_vecs;
    v1 = v1 < P.nvec ? v1 : P.nvec;
    int s = P.tile_seg[tile];
    uint4 x[kPackBatch];
    char* tens[kPackBatch];
    unsigned long long left[kPackBatch];  // valid elements from tens on (>= VEL: full vector)
#pragma unroll
    for (int u = 0; u < kPackBatch; ++u) {
      const unsigned long long v = v0 + (unsigned long long)u * blockDim.x + threadIdx.x;
      left[u] = 0;
      tens[u] = nullptr;
      if (v < v1) {
        if (s < s_hi && P.segs[s + 1].vbeg <= v) s = find_seg(P, v, s, s_hi);
        const unsigned long long e0 = v * VEL - P.segs[s].dst_off;
        const unsigned long long cnt = P.segs[s].count;
        tens[u] = src_tab[s] + e0 * ESZ;
        left[u] = cnt - e0;
        const bool fast = left[u] >= (unsigned long long)VEL && ((reinterpret_cast<uintptr_t>(tens[u]) & 15) == 0);
        if (PACK) {
          if (fast) {
            x[u] = __ldcs(reinterpret_cast<const uint4*>(tens[u]));
          } else {  // ragged member end or misaligned tensor: element by element, zero padding
            alignas(16) char tmp[kPackVecBytes];
#pragma unroll
            for (int i = 0; i < VEL; ++i) {
              if ((unsigned long long)i < left[u]) {
                for (int bb = 0; bb < ESZ; ++bb) tmp[i * ESZ + bb] = tens[u][i * ESZ + bb];
              } else {
                for (int bb = 0; bb < ESZ; ++bb) tmp[i * ESZ + bb] = 0;  // interior padding
              }
            }
            x[u] = *reinterpret_cast<const uint4*>(tmp);
          }
        } else {
          x[u] = __ldcg(reinterpret_cast<const uint4*>(buf + v * kPackVecBytes));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kPackBatch; ++u) {
      const unsigned long long v = v0 + (unsigned long long)u * blockDim.x + threadIdx.x;
      if (v >= v1) continue;
      if (PACK) {
        *reinterpret_cast<uint4*>(buf + v * kPackVecBytes) = Pack16<ESZ>::conv(x[u], P.scale, P.scale_on, dtype);
      } else {
        const bool fast = left[u] >= (unsigned long long)VEL && ((reinterpret_cast<uintptr_t>(tens[u]) & 15) == 0);
        if (fast) {
          __stcs(reinterpret_cast<uint4*>(tens[u]), x[u]);
        } else {
          const char* xb = reinterpret_cast<const char*>(&x[u]);
#pragma unroll
          for (int i = 0; i < VEL; ++i)
            if ((unsigned long long)i < left[u])
              for (int bb = 0; bb < ESZ; ++bb) tens[u][i * ESZ + bb] = xb[i * ESZ + bb];
        }
      }
    }
  }
}

// ------------------------------------------------------------------ fused zero-copy path
// One launch per fusion buffer does Tensor Fusion steps 3-5 and
// the ring without materialising the packed buffer:
//   RS step 0      nscratch <- gather(x) * s                       (pack fused in)
//   RS step s >= 1 nscratch <- gather(x) * s + scratch
//   AG step 0      nbuf     <- gather(x) * s + scratch ; x <- same  (unpack fused in)
//   AG step s >= 1 nbuf     <- buf ; x <- buf
//   final          x <- buf for the chunk received in the last AG step
//   N = 1          x <- gather(x) * s
// gather/scatter map a 16 B buffer vector to its member through the plan's
// segment table (vbeg cached in shared memory).  Every element is gathered
// exactly once before it is scattered (same CTA, program order), so the
// in-place update of the caller's tensors is safe.  Results are bit-identical
// to pack -> ring -> unpack: same per-element operations in the same order.
enum FusedKind { kF_RS0 = 0, kF_RS = 1, kF_AG0 = 2, kF_AG = 3, kF_FIN = 4,
                 kF_RAG0 = 8,   // registered all-gather step 0: final -> own tensors + successor's tensors
                 kF_RAG = 9,    // registered all-gather step s >= 1: own tensors -> successor's tensors
                 kF_G2B = 6,    // broadcast root:        nbuf <- gather(x)
                 kF_G2BS = 7,   // allgather own block:   nbuf <- gather(in); out <- same
                 kF_SOLO = 10 };// N = 1 (bulk kernel): x <- gather(x) * s

struct FusedCtx {
  const PackSeg* segs;
  char* const* src;                 // this rank's gather addresses [nseg]
  char* const* dst;                 // this rank's scatter addresses [nseg] (== src for allreduce)
  char* const* rdst;                // registered mode: the successor's tensor addresses [nseg]
  const unsigned long long* vbeg;   // shared or global copy of segs[].vbeg
  const char* scr;                  // fused ring: this buffer's receive half (own scratch)
  char* nscr;                       //   and the successor's half it pushes into
  int nseg;
  int scale_on;
  float scale;
  int dtype;
  unsigned pace_cyc, pace_burst;    // remote-store pacing (RingParams)
  const int* tile_seg;              // BufDesc::tile_seg when vbeg is in global memory (else nullptr)
  unsigned long long tile_vecs;
};

// Remote-store pacing (HVD_CFG_PACE_GBPS): a channel issues at most one row of remote
// stores per pace_cyc ns, with up to pace_burst ns of credit after idling.
// Keeping the offered NVLink load just under what the link drains keeps the store
// queue — and with it the fence and arrival latency of every ring hop — short.
// Time is %globaltimer (ns), not SM cycles: the SM clock drops under load and differs
// between GPUs, which would pace the ranks of a ring at different real rates.
__device__ __forceinline__ void pace_row(const FusedCtx& F, long long& vft) {
  long long now = (long long)globaltimer();
  const long long start = vft > now - (long long)F.pace_burst ? vft : now - (long long)F.pace_burst;
  vft = start + F.pace_cyc;
  while (now < start) now = (long long)globaltimer();
}

__device__ __forceinline__ int seg_of(const FusedCtx& F, unsigned long long v, int s) {
  if (F.vbeg[s] <= v && (s + 1 == F.nseg || F.vbeg[s + 1] > v)) return s;
  int lo = 0, hi = F.nseg - 1;
  if (F.tile_seg) {  // the plan's tile -> member map narrows the search to a few members
    const unsigned long long p = v / F.tile_vecs;
    lo = __ldg(F.tile_seg + p);
    hi = __ldg(F.tile_seg + p + 1);
  }
  while (lo < hi) {  // largest s with vbeg[s] <= v
    const int mid = (lo + hi + 1) >> 1;
    if (F.vbeg[mid] <= v) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Element-by-element paths (ragged member end, misaligned tensor, tail past the
// last member) are out of line: they are rare and would otherwise inflate the
// register allocation of the vector loop.
template <int ESZ>
__device__ __noinline__ uint4 gather_slow(const char* tp, unsigned long long left) {
  constexpr int VEL = 16 / ESZ;
  alignas(16) char tmp[16];
#pragma unroll
  for (int i = 0; i < VEL; ++i)
#pragma unroll
    for (int b = 0; b < ESZ; ++b) tmp[i * ESZ + b] = (unsigned long long)i < left ? tp[i * ESZ + b] : 0;
  return *reinterpret_cast<const uint4*>(tmp);
}

template <int ESZ>
__device__ __noinline__ void scatter_slow(char* tp, unsigned long long left, uint4 x) {
  constexpr int VEL = 16 / ESZ;
  const char* xb = reinterpret_cast<const char*>(&x);
#pragma unroll
  for (int i = 0; i < VEL; ++i)
    if ((unsigned long long)i < left)
#pragma unroll
      for (int b = 0; b < ESZ; ++b) tp[i * ESZ + b] = xb[i * ESZ + b];
}

// Per-thread cache of the member that owns the current buffer vectors: a slice
// walks long runs of vectors inside one member, so the table lookup (shared
// memory binary search + two global loads) happens once per member per thread.
struct SegCache {
  unsigned long long vlo = 1, vhi = 0;  // vectors [vlo, vhi) belong to member s (empty at start)
  unsigned long long end_el = 0;        // member end, buffer element index
  uintptr_t g = 0, d = 0;               // gather / scatter address of buffer element 0 of this member
  uintptr_t rd = 0;                     // registered mode: successor's address of buffer element 0
  int s = 0;
};

template <int ESZ>
__device__ __forceinline__ void seg_lookup(const FusedCtx& F, unsigned long long v, SegCache& c) {
  if (v >= c.vlo && v < c.vhi) return;
  const int s = seg_of(F, v, c.s);
  c.s = s;
  c.vlo = F.vbeg[s];
  c.vhi = s + 1 < F.nseg ? F.vbeg[s + 1] : ~0ull;
  const unsigned long long dst_off = F.segs[s].dst_off;
  c.end_el = dst_off + F.segs[s].count;
  c.g = reinterpret_cast<uintptr_t>(F.src[s]) - dst_off * ESZ;
  c.d = reinterpret_cast<uintptr_t>(F.dst[s]) - dst_off * ESZ;
  if (F.rdst) c.rd = reinterpret_cast<uintptr_t>(F.rdst[s]) - dst_off * ESZ;
}

// seg_lookup for a vector whose member is among the nc members s0.. whose start vectors
// are staged in shared memory (vb[i] = vbeg[s0 + i]; v < vb[nc - 1] or s0 + nc == nseg).
template <int ESZ>
__device__ __forceinline__ void seg_lookup_staged(const FusedCtx& F, unsigned long long v, SegCache& c,
                                                  const unsigned long long* vb, int s0, int nc) {
  if (v >= c.vlo && v < c.vhi) return;
  int lo = c.s >= s0 && c.s < s0 + nc && vb[c.s - s0] <= v ? c.s - s0 : 0, hi = nc - 1;
  while (lo < hi) {  // largest i with vb[i] <= v
    const int mid = (lo + hi + 1) >> 1;
    if (vb[mid] <= v) lo = mid; else hi = mid - 1;
  }
  const int s = s0 + lo;
  c.s = s;
  c.vlo = vb[lo];
  c.vhi = lo + 1 < nc ? vb[lo + 1] : (s + 1 < F.nseg ? F.vbeg[s + 1] : ~0ull);
  const unsigned long long dst_off = F.segs[s].dst_off;
  c.end_el = dst_off + F.segs[s].count;
  c.g = reinterpret_cast<uintptr_t>(F.src[s]) - dst_off * ESZ;
  c.d = reinterpret_cast<uintptr_t>(F.dst[s]) - dst_off * ESZ;
  if (F.rdst) c.rd = reinterpret_cast<uintptr_t>(F.rdst[s]) - dst_off * ESZ;
}

template <int ESZ>
__device__ __forceinline__ bool fast16(const char* tp, unsigned long long left) {
  return left >= (unsigned long long)(16 / ESZ) && ((reinterpret_cast<uintptr_t>(tp) & 15) == 0);
}

// cp.async (LDGSTS) 16 B global -> shared, L2 only: the slice loop prefetches each
// thread's own future vectors kPipe rows ahead into private shared-memory slots,
// so kPipe x (1-2) x 16 B per thread are in flight without holding registers.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Tensor <-> wire conversion of one 16 B wire vector (R14).  W = wire element
// size, T = tensor element size; TB = tensor bytes per wire vector.  Same
// dtype: plain 16 B (plus the AVERAGE prescale).  fp32 tensor / bf16 wire:
// 32 B of tensor, fl32(x*s) rounded RNE.  bf16 tensor / fp32 wire: 8 B of
// tensor, widened exactly, then fl32(x*s).
struct Raw32 { uint4 a, b; };

template <int W, int T> struct WireCvt;

template <int E> struct WireCvt<E, E> {
  __device__ static __forceinline__ bool fast(const char* p, unsigned long long left) { return fast16<E>(p, left); }
  __device__ static __forceinline__ void issue(Raw32* slot, const char* p) { cp_async16(&slot->a, p); }
  __device__ static __forceinline__ void load(Raw32& r, const char* p) { r.a = __ldcs(reinterpret_cast<const uint4*>(p)); }
  __device__ static __forceinline__ uint4 take(const Raw32& r, float s, int on, int dtype) {
    return Pack16<E>::conv(r.a, s, on, dtype);
  }
  __device__ static __forceinline__ uint4 slow(const char* p, unsigned long long left, float s, int on, int dtype) {
    return Pack16<E>::conv(gather_slow<E>(p, left), s, on, dtype);
  }
  __device__ static __forceinline__ void put(char* p, unsigned long long left, const uint4& x) {
    if (fast16<E>(p, left)) *reinterpret_cast<uint4*>(p) = x;
    else scatter_slow<E>(p, left, x);
  }
};

template <> struct WireCvt<2, 4> {  // fp32 tensor, bf16 wire
  __device__ static __forceinline__ bool fast(const char* p, unsigned long long left) {
    return left >= 8 && ((reinterpret_cast<uintptr_t>(p) & 15) == 0);
  }
  __device__ static __forceinline__ void issue(Raw32* slot, const char* p) {
    cp_async16(&slot->a, p);
    cp_async16(&slot->b, p + 16);
  }
  __device__ static __forceinline__ void load(Raw32& r, const char* p) {
    r.a = __ldcs(reinterpret_cast<const uint4*>(p));
    r.b = __ldcs(reinterpret_cast<const uint4*>(p + 16));
  }
  __device__ static __forceinline__ uint4 pack8(const float (&f)[8], float s, int on) {
    float g[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) g[i] = on ? __fmul_rn(f[i], s) : f[i];
    return make_uint4(pack_bf16x2(g[0], g[1]), pack_bf16x2(g[2], g[3]), pack_bf16x2(g[4], g[5]),
                      pack_bf16x2(g[6], g[7]));
  }
  __device__ static __forceinline__ uint4 take(const Raw32& r, float s, int on, int) {
    const float f[8] = {__uint_as_float(r.a.x), __uint_as_float(r.a.y), __uint_as_float(r.a.z), __uint_as_float(r.a.w),
                        __uint_as_float(r.b.x), __uint_as_float(r.b.y), __uint_as_float(r.b.z), __uint_as_float(r.b.w)};
    return pack8(f, s, on);
  }
  __device__ static __noinline__ uint4 slow(const char* p, unsigned long long left, float s, int on, int) {
    float f[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = (unsigned long long)i < left ? reinterpret_cast<const float*>(p)[i] : 0.f;
    return pack8(f, s, on);
  }
  __device__ static __forceinline__ void put(char* p, unsigned long long left, const uint4& x) {
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
    float f[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = bf16lo(w[i]);
      f[2 * i + 1] = bf16hi(w[i]);
    }
    if (fast(p, left)) {
      reinterpret_cast<float4*>(p)[0] = make_float4(f[0], f[1], f[2], f[3]);
      reinterpret_cast<float4*>(p)[1] = make_float4(f[4], f[5], f[6], f[7]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if ((unsigned long long)i < left) reinterpret_cast<float*>(p)[i] = f[i];
    }
  }
};

template <> struct WireCvt<4, 2> {  // bf16 tensor, fp32 wire
  __device__ static __forceinline__ bool fast(const char* p, unsigned long long left) {
    return left >= 4 && ((reinterpret_cast<uintptr_t>(p) & 7) == 0);
  }
  __device__ static __forceinline__ void issue(Raw32* slot, const char* p) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(&slot->a)),
                 "l"(p) : "memory");
  }
  __device__ static __forceinline__ void load(Raw32& r, const char* p) {
    const uint2 h = __ldcs(reinterpret_cast<const uint2*>(p));
    r.a.x = h.x;
    r.a.y = h.y;
  }
  __device__ static __forceinline__ uint4 widen4(uint32_t lo2, uint32_t hi2, float s, int on) {
    float f[4] = {bf16lo(lo2), bf16hi(lo2), bf16lo(hi2), bf16hi(hi2)};
#pragma unroll
    for (int i = 0; i < 4; ++i) f[i] = on ? __fmul_rn(f[i], s) : f[i];
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
  }
  __device__ static __forceinline__ uint4 take(const Raw32& r, float s, int on, int) { return widen4(r.a.x, r.a.y, s, on); }
  __device__ static __noinline__ uint4 slow(const char* p, unsigned long long left, float s, int on, int) {
    uint16_t h[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = (unsigned long long)i < left ? reinterpret_cast<const uint16_t*>(p)[i] : 0;
    return widen4(uint32_t(h[0]) | (uint32_t(h[1]) << 16), uint32_t(h[2]) | (uint32_t(h[3]) << 16), s, on);
  }
  __device__ static __forceinline__ void put(char* p, unsigned long long left, const uint4& x) {
    const uint32_t a = pack_bf16x2(__uint_as_float(x.x), __uint_as_float(x.y));
    const uint32_t b = pack_bf16x2(__uint_as_float(x.z), __uint_as_float(x.w));
    if (fast(p, left)) {
      *reinterpret_cast<uint2*>(p) = make_uint2(a, b);
    } else {
      const uint16_t h[4] = {uint16_t(a), uint16_t(a >> 16), uint16_t(b), uint16_t(b >> 16)};
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if ((unsigned long long)i < left) reinterpret_cast<uint16_t*>(p)[i] = h[i];
    }
  }
};

// One slice [lo, hi) of the fused kernel by the data threads.  Row j of the
// slice is vector v = v_lo + j*nthr + tid.  slots0/slots1: [kPipe][nthr] uint4.
// Handshake to complete inside a slice (the launch's first remote push): the
// slice's first loads are issued, then the leader waits for the successor's
// ready flag while they fly.
// The fused kernel's wait for the predecessor's counter: through the watcher's shared
// copy when the watcher runs, else a system-scope spin on the counter itself.
__device__ __forceinline__ bool dep_wait(const RingParams& R, const unsigned long long* s_flag,
                                         const unsigned long long* flag, unsigned long long target) {
  if (!R.watcher) return spin_until(flag, target, R.err, R.timeout_ns);
  if (ld_acquire_cta_shared64(s_flag) >= target) return true;
  const unsigned long long t0 = globaltimer();
  unsigned spins = 0;
  while (ld_acquire_cta_shared64(s_flag) < target) {
    if ((++spins & 1023u) == 0) {
      if (globaltimer() - t0 > R.timeout_ns || *(volatile int*)R.err != 0) {
        raise_err(R.err, kHvdErrTimeout);
        return false;
      }
    }
  }
  return true;
}

struct DepWait {  // the ring dependency of a slice, waited for inside fused_slice
  const RingParams* R;
  const unsigned long long* s_flag;  // watcher's shared copy
  const unsigned long long* flag;    // the predecessor's counter
  unsigned long long target;
  int* abort;                        // shared abort flag of the CTA
};

struct Handshake {
  const unsigned long long* flag;  // nullptr: none
  const unsigned long long* hash_flag;  // the successor's call hash, written before its flag
  unsigned long long hash;              // this rank's call hash
  unsigned long long epoch;
  int* err;
  unsigned long long timeout_ns;
  int* abort;                      // shared abort flag of the CTA
};

template <class Op, int KIND, int TESZ = Op::kEsz>
__device__ __forceinline__ void fused_slice(const FusedCtx& F, const RingRank& me, unsigned long long lo,
                                            unsigned long long hi, unsigned tid, unsigned nthr, SegCache& sc,
                                            Raw32* slots0, uint4* slots1, long long pv = 0,
                                            const Handshake* hs = nullptr, long long* vft = nullptr,
                                            const DepWait* dep = nullptr) {
  // pv: shift from a buffer vector index to its slot in the channel-private layout of
  // the scratch / fusion-buffer regions (0: buffer order)
  constexpr int ESZ = Op::kEsz;  // wire element size
  constexpr int VEL = 16 / ESZ;
  using Cvt = WireCvt<ESZ, TESZ>;
  constexpr bool GATHER = KIND == kF_RS0 || KIND == kF_RS || KIND == kF_AG0 ||
                          KIND == kF_G2B || KIND == kF_G2BS || KIND == kF_RAG0 || KIND == kF_RAG;
  constexpr bool SCALE = KIND != kF_RAG;  // the registered forward reads final values: no prescale
  constexpr bool SCATTER = KIND == kF_AG0 || KIND == kF_AG || KIND == kF_FIN || KIND == kF_G2BS ||
                           KIND == kF_RAG0;
  constexpr bool RSCATTER = KIND == kF_RAG0 || KIND == kF_RAG;  // into the successor's tensors
  constexpr bool ADD = KIND == kF_RS || KIND == kF_AG0 || KIND == kF_RAG0;
  constexpr bool TO_NSCRATCH = KIND == kF_RS0 || KIND == kF_RS;
  constexpr bool TO_NBUF = KIND == kF_AG0 || KIND == kF_AG || KIND == kF_G2B || KIND == kF_G2BS;
  const unsigned long long v_lo = lo / VEL;
  const unsigned long long v_hi = (hi + VEL - 1) / VEL;
  if (!hs && !dep && v_hi <= v_lo + tid) return;  // (with a wait inside every thread reaches its barrier)
  const int rows = v_hi <= v_lo + tid ? 0 : (int)((v_hi - v_lo - tid + nthr - 1) / nthr);  // rows this thread owns
  SegCache ci = sc;  // issue-side cache (runs kPipe-1 rows ahead of the consume side)
  auto issue = [&](int j) {
    if (j < rows) {
      const unsigned long long v = v_lo + (unsigned long long)j * nthr + tid;
      Raw32* d0 = slots0 + (j % kPipe) * nthr + tid;
      if (GATHER) {
        seg_lookup<TESZ>(F, v, ci);
        const unsigned long long e = v * VEL;
        const unsigned long long left = ci.end_el > e ? ci.end_el - e : 0;
        const char* tp = reinterpret_cast<const char*>(ci.g + e * TESZ);
        if (Cvt::fast(tp, left)) Cvt::issue(d0, tp);
      } else {
        cp_async16(&d0->a, me.buf + (v + pv) * 16);
      }
      if (ADD) cp_async16(slots1 + (j % kPipe) * nthr + tid, F.scr + (v + pv) * 16);
    }
    cp_async_commit();  // one group per row, possibly empty: keeps wait_group counting uniform
  };
  int nrows = rows;
  if (GATHER && ADD && dep) {
    // the ring dependency is waited for here, after this op's first gradient loads are in
    // flight: only the received partials (scratch) must wait for the predecessor
    auto issue_a = [&](int j) {
      if (j < rows) {
        const unsigned long long v = v_lo + (unsigned long long)j * nthr + tid;
        seg_lookup<TESZ>(F, v, ci);
        const unsigned long long e = v * VEL;
        const unsigned long long left = ci.end_el > e ? ci.end_el - e : 0;
        const char* tp = reinterpret_cast<const char*>(ci.g + e * TESZ);
        if (Cvt::fast(tp, left)) Cvt::issue(slots0 + (j % kPipe) * nthr + tid, tp);
      }
    };
#pragma unroll
    for (int j = 0; j < kPipe - 1; ++j) issue_a(j);  // uncommitted: they join row 0's group
    if (tid == 0 && !*(volatile int*)dep->abort && !dep_wait(*dep->R, dep->s_flag, dep->flag, dep->target))
      *(volatile int*)dep->abort = 1;
    bar_sync(kBarData, nthr);
    if (*(volatile int*)dep->abort) nrows = 0;
#pragma unroll
    for (int j = 0; j < kPipe - 1; ++j) {
      if (j < rows) {
        const unsigned long long v = v_lo + (unsigned long long)j * nthr + tid;
        cp_async16(slots1 + (j % kPipe) * nthr + tid, F.scr + (v + pv) * 16);
      }
      cp_async_commit();
    }
  } else {
#pragma unroll
    for (int j = 0; j < kPipe - 1; ++j) issue(j);
  }
  if (hs) {
    if (tid == 0) {
      if (!spin_until(hs->flag, hs->epoch, hs->err, hs->timeout_ns)) {
        *(volatile int*)hs->abort = 1;
      } else if (*(volatile const unsigned long long*)hs->hash_flag != hs->hash) {  // ordered by the acquire
        raise_err(hs->err, kHvdErrMismatch);
        *(volatile int*)hs->abort = 1;
      }
    }
    bar_sync(kBarData, nthr);
    if (*(volatile int*)hs->abort) nrows = 0;
  }
  for (int j = 0; j < nrows; ++j) {
    issue(j + kPipe - 1);
    cp_async_wait<kPipe - 1>();  // row j has landed in this thread's slots
    const unsigned long long v = v_lo + (unsigned long long)j * nthr + tid;
    unsigned long long left = 0;
    unsigned long long e = v * VEL;
    if (GATHER || SCATTER) {
      seg_lookup<TESZ>(F, v, sc);
      left = sc.end_el > e ? sc.end_el - e : 0;
    }
    uint4 x;
    if (GATHER) {
      const char* gp = reinterpret_cast<const char*>(sc.g + e * TESZ);
      const int on = SCALE ? F.scale_on : 0;
      x = Cvt::fast(gp, left) ? Cvt::take(slots0[(j % kPipe) * nthr + tid], F.scale, on, F.dtype)
                              : Cvt::slow(gp, left, F.scale, on, F.dtype);
    } else {
      x = slots0[(j % kPipe) * nthr + tid].a;
    }
    if (ADD) {
      const uint4 y = slots1[(j % kPipe) * nthr + tid];
      Op::template add_words<4>(reinterpret_cast<uint32_t*>(&x), reinterpret_cast<const uint32_t*>(&y));
    }
    if ((TO_NSCRATCH || TO_NBUF || RSCATTER) && F.pace_cyc) pace_row(F, *vft);
    if (TO_NSCRATCH) *reinterpret_cast<uint4*>(F.nscr + (v + pv) * 16) = x;
    if (TO_NBUF) *reinterpret_cast<uint4*>(me.nbuf + (v + pv) * 16) = x;
    if (SCATTER) Cvt::put(reinterpret_cast<char*>(sc.d + e * TESZ), left, x);
    if (RSCATTER) Cvt::put(reinterpret_cast<char*>(sc.rd + e * TESZ), left, x);
  }
  cp_async_wait<0>();
}

// j-th operation of a fused launch -> (iteration t, slice k).  Iterations
// 0..T-2 come in order; then the last all-gather iteration T-1 and the final
// local scatter T are interleaved with a lag of `lag` slices:
//   AG_0 .. AG_lag, then (FIN_p, AG_{p+lag+1}) for p = 0.., then the remaining FINs
// (lag >= K-1: all AG slices first, then all FIN slices).
__device__ __host__ __forceinline__ void fused_op(int j, int K, int T, int lag, int& t, int& k) {
  const int head = (T - 1) * K;
  if (j < head) {
    t = j / K;
    k = j - t * K;
    return;
  }
  const int m = j - head;
  const int first = lag + 1 < K ? lag + 1 : K;
  if (m < first) {
    t = T - 1;
    k = m;
    return;
  }
  const int q = m - first;
  const int pairs = K - first;  // (FIN, AG) pairs
  if (q < 2 * pairs) {
    const int p = q >> 1;
    if ((q & 1) == 0) { t = T; k = p; } else { t = T - 1; k = p + first; }
  } else {
    t = T;
    k = pairs + (q - 2 * pairs);
  }
}

// Geometry of one slice of buffer D: chunk c, channel ch, slice k -> [lo, hi).
__device__ __forceinline__ void slice_range_d(const BufDesc& D, int c, int ch, int k, unsigned long long& lo,
                                              unsigned long long& hi) {
  const unsigned long long L = D.L;
  unsigned long long c_lo = (unsigned long long)c * D.q;
  c_lo = c_lo < L ? c_lo : L;
  unsigned long long c_hi = c_lo + D.q;
  c_hi = c_hi < L ? c_hi : L;
  unsigned long long h_lo = c_lo + (unsigned long long)ch * D.ch_el;
  h_lo = h_lo < c_hi ? h_lo : c_hi;
  unsigned long long h_hi = h_lo + D.ch_el;
  h_hi = h_hi < c_hi ? h_hi : c_hi;
  lo = h_lo + (unsigned long long)k * D.slice_el;
  lo = lo < h_hi ? lo : h_hi;
  hi = lo + D.slice_el;
  hi = hi < h_hi ? hi : h_hi;
}

// Channel ch's index among the channels of buffer D (D.owner < 0: all of them; else the
// D.nch channels owner, owner+1, ... mod nch), or -1 if it takes no part.
__device__ __forceinline__ int chan_of(const BufDesc& D, int ch, int nch) {
  if (D.owner < 0) return ch;
  const int d = (ch - D.owner + nch) % nch;
  return d < D.nch ? d : -1;
}

// Every fusion buffer of a call (up to kMaxMultiBufs) in ONE persistent launch:
// each channel walks the buffers in order with no grid-wide barrier between
// them, so buffer b+1's first pushes overlap buffer b's tail.  That is safe
// because the scratch and fusion-buffer regions are laid out channel-private
// (slot of element e of chunk c in channel ch = ch*region + c*ch_el + offset):
// only channel ch of the successor ever reads what channel ch writes, and a
// channel finishes buffer b (all of its own reads) before it starts b+1.  Signal
// counters continue across buffers (base of buffer b = base + sum of T*K).
//   registered: the all-gather writes final values into the successor's tensors.
// A launch begins with a handshake (ready flag per channel and epoch) so that no
// push lands in a receive region the successor's previous launch still reads.
template <class Op, int TESZ>
#ifdef HVD_FUSED_MAXNREG  // tuning builds: a register cap instead of the launch bounds
#define HVD_FUSED_BOUNDS __maxnreg__(HVD_FUSED_MAXNREG)
#else
#define HVD_FUSED_BOUNDS __launch_bounds__(416, 1)
#endif
__global__ void HVD_FUSED_BOUNDS fused_allreduce_kernel(const __grid_constant__ FusedParams P) {
  if (P.ring.pdl) {
    // programmatic dependent launch: the next launch on the stream may be scheduled onto
    // SMs as they free up; this grid touches memory only once the previous one has
    // completed (its receive regions are free: the handshake below still means that)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  JtGuard jtg(P.ring.jt);
  extern __shared__ __align__(16) unsigned long long s_dyn[];
  constexpr int VEL = 16 / Op::kEsz;
  const RingParams& R = P.ring;
  const RingRank& me = R.rk[blockIdx.y];
  const int ch = blockIdx.x;
  const int N = R.N;
  const int r = me.rank;
  const unsigned long long base0 = R.base[ch];
  const int T = N > 1 ? 2 * (N - 1) : 0;
  const int nd = blockDim.x - 32 * (R.sig_warps + R.watcher);  // data threads
  __shared__ int s_abort, s_done, s_pub, s_claim;
  __shared__ unsigned long long s_flag;  // watcher: newest value of the predecessor's counter
  unsigned long long* s_vbeg = s_dyn;
  Raw32* slots0 = reinterpret_cast<Raw32*>(s_dyn + P.cache_segs);
  uint4* slots1 = reinterpret_cast<uint4*>(slots0 + kPipe * nd);
  if (threadIdx.x == 0) {
    s_abort = 0;
    s_done = 0;
    s_pub = 0;
    s_claim = 0;
    s_flag = 0;
  }
  __syncthreads();
  if (N == 1) return;  // N = 1 runs solo_kernel
  if (threadIdx.x >= nd) {  // ---- signal warp
    // handshake: this launch started, so this rank's previous launch has finished with
    // its receive regions — the predecessor may push (relaxed: the kernel boundary orders it)
    if (threadIdx.x == nd) {  // the call hash first, then the epoch (release orders the two)
      st_relaxed_sys(me.phash + ch, R.hash);
      st_release_sys(me.pready + ch, R.epoch);
    }
    int total = 0;
    for (int b = 0; b < P.nbuf; ++b)
      if (chan_of(P.bufs[b], ch, gridDim.x) >= 0) total += T * P.bufs[b].K;
    if (R.watcher && threadIdx.x >= blockDim.x - 32) {  // the last warp: the watcher
      if (threadIdx.x != blockDim.x - 32) return;
      // dependency watcher (HVD_CFG_WATCHER): keeps the newest value of the predecessor's
      // counter in shared memory, so the data-warp leader waits on a CTA-scope acquire of
      // shared memory instead of a system-scope load after each slice.  Causality: the
      // predecessor's release (sys) -> this acquire (sys) -> release (cta) -> the leader's
      // acquire (cta) -> bar.sync -> the data warps' loads.
      const unsigned long long need = base0 + (unsigned long long)total;
      unsigned long long seen = 0, t0 = 0;
      unsigned spins = 0;
      while (seen < need) {
        const unsigned long long v = ld_acquire_sys(me.flags + ch);
        if (v != seen) {
          seen = v;
          st_release_cta_shared64(&s_flag, v);
          t0 = 0;
          continue;
        }
        if ((++spins & 1023u) == 0) {
          if (*(volatile int*)&s_abort) break;
          const unsigned long long now = globaltimer();
          if (t0 == 0) t0 = now;
          else if (now - t0 > R.timeout_ns + 1000000000ull) break;  // the leader's watchdog reports it
        }
      }
      return;
    }
    if (R.sig_warps > 1) {
      if ((threadIdx.x - nd) % 32 == 0 && total > 0)
        signal_loop_multi(&s_done, &s_claim, total, me.nflags + ch, base0, &s_pub);
      return;
    }
    if (threadIdx.x == nd && total > 0)
      signal_loop(&s_done, total, me.nflags + ch, base0, R.sig_mode, &s_pub,
                  R.tl ? R.tl + tl_words(R.tl_max) * blockIdx.y + ((size_t)kMaxChannels + ch) * R.tl_max * 2 : nullptr,
                  R.tl_max);
    return;
  }
  unsigned long long* tl_d = R.tl ? R.tl + tl_words(R.tl_max) * blockIdx.y + (size_t)ch * R.tl_max * 2 : nullptr;
  int nrec = 0;
  const unsigned tid = threadIdx.x;
  unsigned long long sent = 0;
  int i = 0;                         // ring ops published so far (all buffers)
  unsigned long long bbase = base0;  // counter base of the current buffer
  bool first = true;
  int bpar = 0;  // receive half of this channel's next buffer
  // the launch's first remote push waits for the successor's handshake (inside the slice,
  // after its first loads are issued)
  const Handshake hs0 = {me.rflags + ch, me.rhash + ch, R.hash, R.epoch, R.err, R.timeout_ns, &s_abort};
  bool hs_pending = true;
  long long vft = 0;  // pacing: virtual finish time of this thread's last paced row
  unsigned long long dep_next = 0;  // PREISSUE: the next op's dependency, waited for in its slice
  for (int b = 0; b < P.nbuf; ++b) {
    const BufDesc& D = P.bufs[b];
    const int cg = chan_of(D, ch, gridDim.x);  // this channel's index in the buffer's geometry
    if (cg < 0) continue;                       // a buffer run by other channels
    const int K = D.K;
    const bool cache = D.nseg <= P.cache_segs;
    if (!first) bar_sync(kBarData, nd);  // every data warp is done with the previous member table
    first = false;
    if (cache)
      for (int j = tid; j < D.nseg; j += nd) s_vbeg[j] = D.vbeg[j];
    bar_sync(kBarData, nd);
    FusedCtx F = {};
    F.segs = D.segs;
    F.src = D.src + (size_t)blockIdx.y * D.nseg;
    F.dst = D.dst + (size_t)blockIdx.y * D.nseg;
    F.rdst = P.registered ? D.rdst + (size_t)blockIdx.y * D.nseg : nullptr;
    F.vbeg = cache ? s_vbeg : D.vbeg;
    F.tile_seg = cache ? nullptr : D.tile_seg;
    F.tile_vecs = D.tile_vecs;
    F.nseg = D.nseg;
    F.scale_on = P.scale_on;
    F.scale = P.scale;
    F.dtype = P.dtype;
    F.pace_cyc = R.pace_cyc;
    F.pace_burst = R.pace_burst;
    // Receive halves alternate buffer by buffer on a channel: the predecessor may start
    // buffer b+1 (its reduce-scatter pushes) while this rank still reads buffer b's last
    // partials — registered mode has no final scatter to hold it back — but it cannot
    // start b+2 before this rank's reduce-scatter of b+1, i.e. after b is done here.
    F.scr = bpar ? me.scratch1 : me.scratch;
    F.nscr = bpar ? me.nscratch1 : me.nscratch;
    bpar ^= 1;
    SegCache sc;
    const int nops = P.registered ? T * K : (T + 1) * K;
    for (int j = 0; j < nops; ++j) {
      int t, k;
      if (P.registered) {
        t = j / K;
        k = j - t * K;
      } else {
        fused_op(j, K, T, R.fin_lag, t, k);
      }
      const bool rs = t < N - 1;
      const int s = rs ? t : t - (N - 1);
      const int c = t == T ? mod(r + 2, N) : (rs ? mod(r - s, N) : mod(r + 1 - s, N));
      unsigned long long lo, hi;
      slice_range_d(D, c, cg, k, lo, hi);
      // channel-private slot of this slice's first element, as a vector shift
      const long long pv =
          (long long)(((unsigned long long)ch * P.region_el + (unsigned long long)c * D.ch_el +
                       (lo - (unsigned long long)c * D.q - (unsigned long long)cg * D.ch_el)) / VEL) -
          (long long)(lo / VEL);
      if (R.window > 0 && t < T && i + 1 > R.window) {  // at most `window` pushed-unpublished ops
        if (tid == 0)
          while (ld_acquire_cta_shared(&s_pub) < i + 1 - R.window) __nanosleep(32);
        bar_sync(kBarData, nd);
      }
      const unsigned long long tb = tl_d ? globaltimer() : 0;
      const DepWait dw = {&R, &s_flag, me.flags + ch, dep_next, &s_abort};
      const DepWait* dep = dep_next ? &dw : nullptr;
      if (dep && !(hi > lo && !s_abort)) {  // no data here: the wait still orders this op
        if (tid == 0 && !s_abort && !dep_wait(R, &s_flag, me.flags + ch, dep_next)) s_abort = 1;
        bar_sync(kBarData, nd);
      }
      dep_next = 0;
      if (hi > lo && !s_abort) {
        const Handshake* hs = nullptr;
        if (hs_pending && t < T) {  // every op but the final local scatter pushes
          hs = &hs0;
          hs_pending = false;
        }
        if (P.registered) {
          if (rs && s == 0) fused_slice<Op, kF_RS0, TESZ>(F, me, lo, hi, tid, nd, sc, slots0, slots1, pv, hs, &vft);
          else if (rs) fused_slice<Op, kF_RS, TESZ>(F, me, lo, hi, tid, nd, sc, slots0, slots1, pv, hs, &vft, dep);
          else if (s == 0) fused_slice<Op, kF_RAG0, TESZ>(F, me, lo, hi, tid, nd, sc, slots0, slots1, pv, hs, &vft, dep);
          else fused_slice<Op, kF_RAG, TESZ>(F, me, lo, hi, tid, nd, sc, slots0, slots1, pv, hs, &vft);
        } else {
          if (t == T) fused_slice<Op, kF_FIN, TESZ>(F, me, lo, hi, tid, nd, sc, slots0, slots1, pv);
          else if (rs && s == 0) fused_slice<Op, kF_RS0, TESZ>(F, me, lo, hi, tid, nd, sc, slots0, slots1, pv, hs, &vft);
          else if (rs) fused_slice<Op, kF_RS, TESZ>(F, me, lo, hi, tid, nd, sc, slots0, slots1, pv, hs, &vft, dep);
          else if (s == 0) fused_slice<Op, kF_AG0, TESZ>(F, me, lo, hi, tid, nd, sc, slots0, slots1, pv, hs, &vft, dep);
          else fused_slice<Op, kF_AG, TESZ>(F, me, lo, hi, tid, nd, sc, slots0, slots1, pv, hs, &vft);
        }
        if (t < T) sent += (hi - lo) * Op::kEsz;
      }
      // retire op j (publish it if it is a ring iteration), then wait for op j+1's
      // dependency — the predecessor's (t'-1, k') of the same buffer; publishing first
      // keeps the ring acyclic.  The next buffer's first op (t = 0) has none.
      bar_sync(kBarData, nd);
      if (tl_d && tid == 0 && nrec < R.tl_max) {
        tl_d[2 * nrec] = tb;
        tl_d[2 * nrec + 1] = globaltimer();
        ++nrec;
      }
      if (t < T) ++i;
      int tn = 0, kn = 0;
      if (j + 1 < nops) {
        if (P.registered) {
          tn = (j + 1) / K;
          kn = (j + 1) - tn * K;
        } else {
          fused_op(j + 1, K, T, R.fin_lag, tn, kn);
        }
      }
      const unsigned long long target = tn > 0 ? bbase + (unsigned long long)(tn - 1) * K + kn + 1 : 0;
      // HVD_CFG_PREISSUE: an op that gathers the local gradient and adds the received partial
      // waits for its dependency inside the slice, after its first gradient loads are issued
      const bool inslice = R.preissue && target && tn <= N - 1;
      if (tid == 0) {
        if (t < T) st_release_cta_shared(&s_done, i);
        if (target && !inslice && !s_abort && !dep_wait(R, &s_flag, me.flags + ch, target)) s_abort = 1;
      }
      if (tn > 0 && !inslice) bar_sync(kBarData, nd);
      dep_next = inslice ? target : 0;
    }
    bbase += (unsigned long long)T * K;
  }
  if (tid == 0) {
    // registered: the predecessor's last all-gather slices land in this rank's tensors;
    // completion on the stream means they have arrived
    if (P.registered && N > 1 && !s_abort) dep_wait(R, &s_flag, me.flags + ch, bbase);
    atomicAdd(me.stats + 0, sent);
    if (ch == 0) atomicAdd(me.stats + 1, (unsigned long long)T * P.nbuf);  // messages per buffer
  }
}

// ------------------------------------------------------------------ broadcast / allgather
// Copy collectives on the same machinery (fused_slice, counters, signal warp).
//   broadcast: pipelined ring forward of the root's fusion buffer:
//     root: nbuf <- gather(x); middle ranks: nbuf <- buf, x <- buf; the rank
//     before the root: x <- buf.  One signal per slice on every rank.
//   allgather (R12): ring all-gather of one block per rank (block b at b*q):
//     t = 0: nbuf[r] <- in, out[r] <- in; t >= 1: nbuf[r-t] <- buf, out[r-t] <- buf;
//     final: out[r+1] <- buf.  (N-1)K signals.
// Unlike the allreduce, a rank's first write into its successor's fusion buffer
// can race with the successor still reading that buffer for the previous
// collective, so each launch starts with a handshake: every channel writes
// "ready for epoch e" into its predecessor's ready flag, and waits for its
// successor's before its first remote store.
template <class Op>
__global__ void __launch_bounds__(416, 1) copy_collective_kernel(const __grid_constant__ FusedParams P) {
  JtGuard jtg(P.ring.jt);
  extern __shared__ __align__(16) unsigned long long s_dyn[];
  const RingParams& R = P.ring;
  const RingRank& me = R.rk[blockIdx.y];
  const int ch = blockIdx.x;
  const int N = R.N;
  const int r = me.rank;
  const int K = R.K;
  const unsigned long long base = R.base[ch];
  const bool bcast = R.mode == kRingBroadcast;
  const int T = N - 1;  // allgather ring iterations
  const int nsig = bcast ? K : T * K;
  const int nd = blockDim.x - 32;
  __shared__ int s_abort, s_done, s_pub;
  const bool cache = P.nseg <= kFusedSmemSegs;
  unsigned long long* s_vbeg = s_dyn;
  Raw32* slots0 = reinterpret_cast<Raw32*>(s_dyn + (cache ? (P.nseg + 1) / 2 * 2 : 0));
  uint4* slots1 = reinterpret_cast<uint4*>(slots0 + kPipe * nd);
  if (cache)
    for (int j = threadIdx.x; j < P.nseg; j += blockDim.x) s_vbeg[j] = P.segs[j].vbeg;
  if (threadIdx.x == 0) {
    s_abort = 0;
    s_done = 0;
    s_pub = 0;
    st_release_sys(me.pready + ch, R.epoch);  // this rank's buffers are free for this launch
  }
  __syncthreads();
  if (threadIdx.x >= nd) {
    if (threadIdx.x == nd) signal_loop(&s_done, nsig, me.nflags + ch, base, R.sig_mode, &s_pub);
    return;
  }
  FusedCtx F = {};
  F.segs = P.segs;
  F.src = P.src + (size_t)blockIdx.y * P.nseg;
  F.dst = (P.dst ? P.dst : P.src) + (size_t)blockIdx.y * P.nseg;
  F.rdst = nullptr;
  F.vbeg = cache ? s_vbeg : P.vbeg_global;
  F.nseg = P.nseg;
  F.scale_on = 0;
  F.scale = 1.0f;
  F.dtype = P.dtype;
  const unsigned tid = threadIdx.x;
  SegCache sc;
  unsigned long long sent = 0;
  bool ready = false;  // successor's handshake seen
  const int d = mod(r - R.root, N);  // broadcast: distance from the root
  const int nops = bcast ? K : (T + 1) * K;
  int i = 0;
  for (int j = 0; j < nops; ++j) {
    int t, k, c, kind;
    if (bcast) {
      t = 0;
      k = j;
      c = 0;
      kind = d == 0 ? kF_G2B : (d == N - 1 ? kF_FIN : kF_AG);
    } else {
      fused_op(j, K, T, R.fin_lag, t, k);
      c = t == T ? mod(r + 1, N) : mod(r - t, N);
      kind = t == T ? kF_FIN : (t == 0 ? kF_G2BS : kF_AG);
    }
    const bool remote = kind != kF_FIN;
    // dependency: the predecessor's slice (broadcast: same k; allgather: (t-1, k))
    unsigned long long target = 0;
    if (bcast && d > 0) target = base + (unsigned long long)k + 1;
    if (!bcast && t > 0) target = base + (unsigned long long)(t - 1) * K + k + 1;
    if (tid == 0 && !s_abort) {
      if (target && !spin_until(me.flags + ch, target, R.err, R.timeout_ns)) s_abort = 1;
      if (remote && !ready && !s_abort && !spin_until(me.rflags + ch, R.epoch, R.err, R.timeout_ns)) s_abort = 1;
    }
    if (remote) ready = true;
    bar_sync(kBarData, nd);
    unsigned long long lo, hi;
    slice_range(R, c, ch, k, lo, hi);
    if (hi > lo && !s_abort) {
      if (kind == kF_G2B) fused_slice<Op, kF_G2B>(F, me, lo, hi, tid, nd, sc, slots0, slots1);
      else if (kind == kF_G2BS) fused_slice<Op, kF_G2BS>(F, me, lo, hi, tid, nd, sc, slots0, slots1);
      else if (kind == kF_AG) fused_slice<Op, kF_AG>(F, me, lo, hi, tid, nd, sc, slots0, slots1);
      else fused_slice<Op, kF_FIN>(F, me, lo, hi, tid, nd, sc, slots0, slots1);
      if (remote) sent += (hi - lo) * Op::kEsz;
    }
    bar_sync(kBarData, nd);
    // every ring iteration (broadcast: every slice, even without data) is signalled
    if (bcast || t < T) {
      ++i;
      if (tid == 0) st_release_cta_shared(&s_done, i);
    }
  }
  if (tid == 0) {
    atomicAdd(me.stats + 0, sent);
    if (ch == 0) atomicAdd(me.stats + 1, (unsigned long long)(bcast ? (d == N - 1 ? 0 : 1) : T));
  }
}

// ------------------------------------------------------------------ pull-mode fused allreduce
// Same ring, same reduction order, but every transfer is initiated by the
// RECEIVER: rank r TMA-loads (cp.async.bulk, mbarrier transaction counts) its
// predecessor's partial of chunk c straight from the predecessor's HBM into
// shared memory, adds its own gathered contribution and writes the result into
// ITS OWN pull buffer, where the successor will load it from.  A rank therefore
// never stores to a peer: publishing "slice done" only needs a system fence over
// its LOCAL stores, which is short, whereas a fence behind a stream of NVLink
// stores waits for that whole backlog to drain (tools/fence_probe.cu).
//
// Steps t = 0..2N-2 per slice k (op j = t*K + k, published as base + j + 1):
//   t = 0          B[r]     <- gather(x)*s                          (local)
//   1 <= t <= N-1  B[r-t]   <- pred.B[r-t] + gather(x)*s           (t = N-1: the owner's final
//                                                                   chunk r+1, also scattered)
//   N <= t <= 2N-2 x[c]     <- pred.B[c], c = r+1-(t-N+1); B[c] <- same unless t = 2N-2
// Op (t, k) depends on the predecessor's op (t-1, k).  The pull buffers are
// double-buffered by call parity; before writing buffer p in call k a rank waits
// until its successor has completed call k-2 (the last reader of that buffer).
constexpr int kStageBytes = 16 << 10;
constexpr int kStages = 6;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load(void* smem_dst, const void* gmem_src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(smem_dst)), "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ int pull_chunk(int t, int r, int N) {
  return t < N ? mod(r - t, N) : mod(r + 1 - (t - N + 1), N);
}

template <class Op>
__global__ void __launch_bounds__(416, 1) pull_allreduce_kernel(const __grid_constant__ FusedParams P) {
  JtGuard jtg(P.ring.jt);
  extern __shared__ __align__(128) unsigned long long s_dyn_pull[];  // (own name: 128 B alignment)
  __shared__ __align__(8) unsigned long long full_bar[kStages], empty_bar[kStages];
  __shared__ int s_abort;
  constexpr int ESZ = Op::kEsz;
  constexpr int VEL = 16 / ESZ;
  const RingParams& R = P.ring;
  const RingRank& me = R.rk[blockIdx.y];
  const int ch = blockIdx.x;
  const int N = R.N;
  const int r = me.rank;
  const int K = R.K;
  const unsigned long long base = R.base[ch];
  const int T = 2 * N - 1;
  const int nops = T * K;
  const int nd = blockDim.x - 32;
  const int par = R.parity;
  char* const myB = me.pull[par];
  const char* const predB = me.ppull[par];
  const bool cache = P.nseg <= kFusedSmemSegs;
  unsigned long long* s_vbeg = s_dyn_pull;
  char* stages = reinterpret_cast<char*>(s_dyn_pull + (cache ? (P.nseg + 15) / 16 * 16 : 0));
  if (cache)
    for (int j = threadIdx.x; j < P.nseg; j += blockDim.x) s_vbeg[j] = P.segs[j].vbeg;
  if (threadIdx.x == 0) {
    s_abort = 0;
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], nd / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  unsigned long long* tl_d =
      R.tl ? R.tl + tl_words(R.tl_max) * blockIdx.y + (size_t)ch * R.tl_max * 2 : nullptr;
  if (threadIdx.x >= nd) {  // ---- loader warp: remote polls + TMA loads of the predecessor's buffer
    if (threadIdx.x != nd) return;
    unsigned long long* tl_s =
        R.tl ? R.tl + tl_words(R.tl_max) * blockIdx.y + ((size_t)kMaxChannels + ch) * R.tl_max * 2 : nullptr;
    int nrec = 0;
    unsigned long long seq = 0;
    bool abort = false;
    for (int j = 0; j < nops; ++j) {
      const int t = j / K, k = j - (j / K) * K;
      if (t == 0) continue;
      unsigned long long lo, hi;
      slice_range(R, pull_chunk(t, r, N), ch, k, lo, hi);
      if (!abort && hi > lo) {
        if (!spin_until(me.pflags_pred + ch, base + (unsigned long long)(t - 1) * K + k + 1, R.err, R.timeout_ns)) {
          abort = true;
          s_abort = 1;
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");  // acquire before the async-proxy loads
        if (tl_s && nrec < R.tl_max) {  // timeline: when the predecessor's slice became loadable
          tl_s[2 * nrec] = globaltimer();
          tl_s[2 * nrec + 1] = (unsigned long long)j;
          ++nrec;
        }
      }
      const unsigned long long bytes = hi > lo ? ((hi - lo) * ESZ + 15) / 16 * 16 : 0;
      for (unsigned long long off = 0; off < bytes; off += kStageBytes, ++seq) {
        const int st = (int)(seq % kStages);
        if (seq >= (unsigned long long)kStages) mbar_wait(&empty_bar[st], (unsigned)((seq / kStages - 1) & 1));
        const unsigned pb = (unsigned)(bytes - off < (unsigned long long)kStageBytes ? bytes - off : kStageBytes);
        if (abort) {
          mbar_arrive(&full_bar[st]);  // complete the phase without data so the compute warps move on
        } else {
          mbar_expect_tx(&full_bar[st], pb);
          tma_load(stages + (size_t)st * kStageBytes, predB + lo * ESZ + off, pb, &full_bar[st]);
        }
      }
    }
    return;
  }

  // ---- compute warps
  FusedCtx F = {};
  F.segs = P.segs;
  F.src = P.src + (size_t)blockIdx.y * P.nseg;
  F.dst = (P.dst ? P.dst : P.src) + (size_t)blockIdx.y * P.nseg;
  F.rdst = nullptr;
  F.vbeg = cache ? s_vbeg : P.vbeg_global;
  F.nseg = P.nseg;
  F.scale_on = P.scale_on;
  F.scale = P.scale;
  F.dtype = P.dtype;
  const unsigned tid = threadIdx.x;
  const int lane = tid & 31;
  SegCache sc;
  unsigned long long sent = 0;
  // WAR handshake on the double-buffered pull buffer (see above)
  if (tid == 0 && R.call >= 3 &&
      !spin_until(me.done_succ, (unsigned long long)(R.call - 2), R.err, R.timeout_ns))
    s_abort = 1;
  bar_sync(kBarData, nd);
  unsigned long long seq = 0;
  for (int j = 0; j < nops; ++j) {
    const unsigned long long tb = tl_d ? globaltimer() : 0;
    const int t = j / K, k = j - (j / K) * K;
    const int c = pull_chunk(t, r, N);
    const bool gathers = t <= N - 1;
    const bool scatters = t >= N - 1;
    const bool writes = t <= T - 2;
    unsigned long long lo, hi;
    slice_range(R, c, ch, k, lo, hi);
    const unsigned long long v_lo = lo / VEL, v_hi = (hi + VEL - 1) / VEL;
    if (t == 0) {
      // own contribution of chunk r into the local pull buffer
      if (hi > lo && !s_abort) {
        constexpr int U = 8;  // loads in flight per thread (this step is a local HBM copy)
        for (unsigned long long v0 = v_lo + tid; v0 < v_hi; v0 += (unsigned long long)nd * U) {
          uint4 x[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const unsigned long long v = v0 + (unsigned long long)u * nd;
            if (v < v_hi) {
              seg_lookup<ESZ>(F, v, sc);
              const unsigned long long e = v * VEL;
              const unsigned long long left = sc.end_el > e ? sc.end_el - e : 0;
              const char* gp = reinterpret_cast<const char*>(sc.g + e * ESZ);
              x[u] = fast16<ESZ>(gp, left) ? __ldcs(reinterpret_cast<const uint4*>(gp)) : gather_slow<ESZ>(gp, left);
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const unsigned long long v = v0 + (unsigned long long)u * nd;
            if (v < v_hi)
              *reinterpret_cast<uint4*>(myB + v * 16) = Pack16<ESZ>::conv(x[u], F.scale, F.scale_on, F.dtype);
          }
        }
      }
    } else if (hi > lo) {
      const unsigned long long bytes = ((hi - lo) * ESZ + 15) / 16 * 16;
      for (unsigned long long off = 0; off < bytes; off += kStageBytes, ++seq) {
        const int st = (int)(seq % kStages);
        const unsigned long long pv0 = v_lo + off / 16;
        unsigned long long pv1 = pv0 + kStageBytes / 16;
        pv1 = pv1 < v_hi ? pv1 : v_hi;
        constexpr int kMaxPer = (kStageBytes / 16 + 255) / 256;  // vectors per thread per stage (nd >= 256)
        uint4 g[kMaxPer];
        if (gathers && !s_abort) {  // local gathers issued before waiting for the remote stage
#pragma unroll
          for (int i = 0; i < kMaxPer; ++i) {
            const unsigned long long v = pv0 + tid + (unsigned long long)i * nd;
            if (v < pv1) {
              seg_lookup<ESZ>(F, v, sc);
              const unsigned long long e = v * VEL;
              const unsigned long long left = sc.end_el > e ? sc.end_el - e : 0;
              const char* gp = reinterpret_cast<const char*>(sc.g + e * ESZ);
              g[i] = fast16<ESZ>(gp, left) ? __ldcs(reinterpret_cast<const uint4*>(gp)) : gather_slow<ESZ>(gp, left);
            }
          }
        }
        mbar_wait(&full_bar[st], (unsigned)((seq / kStages) & 1));
        if (!s_abort) {
          const uint4* stg = reinterpret_cast<const uint4*>(stages + (size_t)st * kStageBytes);
#pragma unroll
          for (int i = 0; i < kMaxPer; ++i) {
            const unsigned long long v = pv0 + tid + (unsigned long long)i * nd;
            if (v < pv1) {
              uint4 x = stg[v - pv0];
              if (gathers) {
                const uint4 y = Pack16<ESZ>::conv(g[i], F.scale, F.scale_on, F.dtype);
                Op::template add_words<4>(reinterpret_cast<uint32_t*>(&x), reinterpret_cast<const uint32_t*>(&y));
              }
              if (writes) *reinterpret_cast<uint4*>(myB + v * 16) = x;
              if (scatters) {
                seg_lookup<ESZ>(F, v, sc);
                const unsigned long long e = v * VEL;
                const unsigned long long left = sc.end_el > e ? sc.end_el - e : 0;
                char* tp = reinterpret_cast<char*>(sc.d + e * ESZ);
                if (fast16<ESZ>(tp, left)) *reinterpret_cast<uint4*>(tp) = x;
                else scatter_slow<ESZ>(tp, left, x);
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[st]);
      }
    }
    // traffic stats count what the successor pulls from this rank: the ops that write B
    if (writes && hi > lo) sent += (hi - lo) * ESZ;
    // op j done: publish it (the fence covers this rank's local stores only)
    bar_sync(kBarData, nd);
    if (tid == 0) {
      if (writes) asm volatile("fence.acq_rel.sys;" ::: "memory");
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(me.pflags_own + ch),
                   "l"(base + (unsigned long long)j + 1) : "memory");
      if (tl_d && j < R.tl_max) {
        tl_d[2 * j] = tb;
        tl_d[2 * j + 1] = globaltimer();
      }
    }
  }
  if (tid == 0) {
    atomicAdd(me.stats + 0, sent);
    if (ch == 0) atomicAdd(me.stats + 1, (unsigned long long)(2 * (N - 1)));
    // last CTA of this rank to finish publishes "call done" (its pulls from the predecessor are over)
    const unsigned long long prev = atomicAdd(me.exits, 1ull);
    if (prev + 1 == R.exits_target) st_release_sys(me.done_own, (unsigned long long)R.call);
  }
}

// ------------------------------------------------------------------ LL (low-latency) small-buffer ring
// For small buffers the ring is latency-bound: each of the 2(N-1) steps of the
// store+fence+counter protocol costs a system fence, a counter hop and a
// barrier.  Here every 4 B of wire data travels in one 8 B word together with
// the call's epoch as a flag ({epoch, data}, aligned 8 B stores are single-copy
// atomic), so a receiver polls the data itself: no fences, no counters, no
// barriers — each thread only waits for the words it consumes.  Same ring, same
// chunks, same reduction order as the fused kernel (bit-identical); the wire
// carries 2x the bytes, which does not matter at these sizes.
// LL region of a rank: two fixed halves (parity = epoch & 1), each [step 2N-2][chunk
// slot q] words, written by the predecessor.  A sender reuses a parity two launches
// later, when (stream order + the all-gather chain) its successor has finished with
// it; the halves are fixed so that launches of different sizes never overlap.
#ifndef HVD_LL_BACKOFF
#define HVD_LL_BACKOFF 0
#endif
__device__ __forceinline__ void ll_store(unsigned long long* p, uint4 x, unsigned flag) {
  const unsigned long long f = (unsigned long long)flag << 32;
  asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1,%2};" ::"l"(p), "l"(f | x.x), "l"(f | x.y) : "memory");
  asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1,%2};" ::"l"(p + 2), "l"(f | x.z), "l"(f | x.w) : "memory");
}

// Wait until the 4 words of one data vector carry `flag`; false on watchdog timeout.
__device__ __forceinline__ bool ll_load(const unsigned long long* p, unsigned flag, uint4& x, int* err,
                                        unsigned long long timeout_ns) {
  unsigned long long a, b, c, d;
  unsigned long long t0 = 0;
  unsigned spins = 0;
  for (;;) {
    asm volatile("ld.relaxed.sys.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
    asm volatile("ld.relaxed.sys.global.v2.u64 {%0,%1}, [%2];" : "=l"(c), "=l"(d) : "l"(p + 2) : "memory");
    if ((unsigned)(a >> 32) == flag && (unsigned)(b >> 32) == flag && (unsigned)(c >> 32) == flag &&
        (unsigned)(d >> 32) == flag)
      break;
    if ((++spins & 255u) == 0) {
      const unsigned long long now = globaltimer();
      if (t0 == 0) t0 = now;
      else if (now - t0 > timeout_ns || *(volatile int*)err != 0) {
        raise_err(err, kHvdErrTimeout);
        return false;
      }
    }
#if HVD_LL_BACKOFF > 0
    if (spins > 8) __nanosleep(HVD_LL_BACKOFF);  // fewer polls in flight while the words travel
#endif
  }
  x = make_uint4((uint32_t)a, (uint32_t)b, (uint32_t)c, (uint32_t)d);
  return true;
}

template <class Op>
__global__ void __launch_bounds__(256) ll_allreduce_kernel(const __grid_constant__ FusedParams P) {
  if (P.ring.ll_pdl) {  // HVD_CFG_LL_PDL: the next launch may be scheduled; memory after the previous grid
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  JtGuard jtg(P.ring.jt);
  constexpr int ESZ = Op::kEsz;
  constexpr int VEL = 16 / ESZ;
  const RingParams& R = P.ring;
  const RingRank& me = R.rk[blockIdx.y];
  int ch = blockIdx.x;  // -> (buffer b, channel ch of b): the buffers of a call share one launch
  int b = 0;
  while (b + 1 < P.nbuf && ch >= P.bufs[b].nch) ch -= P.bufs[b++].nch;
  const int N = R.N;
  const int r = me.rank;
  const int T = 2 * (N - 1);
  const BufDesc& D = P.bufs[b];
  const unsigned flag = (unsigned)R.epoch;
  const int par = (int)(R.epoch & 1);
  const unsigned long long slot_words = D.q / VEL * 4;  // words per chunk slot
  // each parity owns a FIXED half of the LL area: a launch of another size must not reach
  // into the other parity, which the successor may still be reading (previous launch)
  constexpr unsigned long long kHalfWords = kLLHalfBytes / 8;
  unsigned long long* const in_ll = me.ll + (unsigned long long)par * kHalfWords + D.ll_off;
  unsigned long long* const out_ll = me.nll + (unsigned long long)par * kHalfWords + D.ll_off;
  FusedCtx F = {};
  F.segs = D.segs;
  F.src = D.src + (size_t)blockIdx.y * D.nseg;
  F.dst = D.dst + (size_t)blockIdx.y * D.nseg;
  F.rdst = nullptr;
  F.vbeg = D.vbeg;
  F.tile_seg = D.tile_seg;
  F.tile_vecs = D.tile_vecs;
  F.nseg = D.nseg;
  F.scale_on = P.scale_on;
  F.scale = P.scale;
  F.dtype = P.dtype;
  using Cvt = WireCvt<ESZ, ESZ>;
  SegCache sc;
  bool ok = true;
  unsigned long long sent = 0;
  for (int t = 0; t <= T && ok; ++t) {  // t == T: the chunk received in the last step
    const bool rs = t < N - 1;
    const int s = rs ? t : t - (N - 1);
    const int c = t == T ? mod(r + 2, N) : (rs ? mod(r - s, N) : mod(r + 1 - s, N));
    unsigned long long lo, hi;
    slice_range_d(D, c, ch, 0, lo, hi);  // one slice per channel (K = 1)
    if (hi <= lo) continue;
    const unsigned long long c0 = (unsigned long long)c * D.q;  // chunk start: slot position base
    const unsigned long long v_lo = lo / VEL, v_hi = (hi + VEL - 1) / VEL;
    for (unsigned long long v = v_lo + threadIdx.x; v < v_hi; v += blockDim.x) {
      const unsigned long long e = v * VEL;
      const unsigned long long slot = (v - c0 / VEL) * 4;  // word offset inside the chunk slot
      unsigned long long left = 0;
      seg_lookup<ESZ>(F, v, sc);
      left = sc.end_el > e ? sc.end_el - e : 0;
      uint4 g = make_uint4(0, 0, 0, 0);
      if (t <= N - 1) {  // own contribution, loaded before polling the predecessor's words
        const char* gp = reinterpret_cast<const char*>(sc.g + e * ESZ);
        g = Cvt::fast(gp, left) ? Pack16<ESZ>::conv(__ldcs(reinterpret_cast<const uint4*>(gp)), F.scale, F.scale_on,
                                                    F.dtype)
                                : Cvt::slow(gp, left, F.scale, F.scale_on, F.dtype);
      }
      uint4 x = g;
      if (t > 0) {
        uint4 in;
        if (!ll_load(in_ll + (unsigned long long)(t - 1) * slot_words + slot, flag, in, R.err, R.timeout_ns)) {
          ok = false;
          break;
        }
        x = in;
        if (t <= N - 1) Op::template add_words<4>(reinterpret_cast<uint32_t*>(&x), reinterpret_cast<const uint32_t*>(&g));
      }
      if (t < T) ll_store(out_ll + (unsigned long long)t * slot_words + slot, x, flag);
      if (t >= N - 1) Cvt::put(reinterpret_cast<char*>(sc.d + e * ESZ), left, x);
    }
    if (t < T) sent += (hi - lo) * ESZ;
  }
  if (threadIdx.x == 0) {
    atomicAdd(me.stats + 0, sent);
    if (ch == 0) atomicAdd(me.stats + 1, (unsigned long long)T);
  }
}

// LL128 protocol: like LL, the data carries its own arrival flag, but per 128-byte
// line instead of per 8-byte word.  An 8-lane group stores a line with ONE warp store
// instruction (16 B per lane); lane 7's second 8 B are the flag {~epoch}; the receiver
// loads the line the same way and accepts it when the flag matches.  This relies on
// NVLink (and L2) delivering one warp store of a 128-byte line whole — what NCCL's
// LL128 also relies on; PTX does not promise it, so hvd_connect enables LL128 only after
// a self-test of exactly this store pattern passes on every rank.  Wire bytes are 16/15
// of the data (lane 7's first 8 B carry data: a pair of lines holds 15 vectors); LL: 2x.
// Same chunks, same reduction order as the ring: bit-identical.
// A half vector (8 B: VEL/2 elements) of an LL128 line's last lane: `left` valid
// elements, placed in x.x / x.y.
template <int ESZ>
__device__ __forceinline__ void put_half(char* p, unsigned long long left, const uint4& x) {
  constexpr int HV = 8 / ESZ;
  if (left >= (unsigned long long)HV && (reinterpret_cast<uintptr_t>(p) & 7) == 0)
    *reinterpret_cast<uint2*>(p) = make_uint2(x.x, x.y);
  else
    scatter_slow<ESZ>(p, left < (unsigned long long)HV ? left : HV, x);
}

template <class Op>
__global__ void __launch_bounds__(256) ll128_allreduce_kernel(const __grid_constant__ FusedParams P) {
  if (P.ring.ll_pdl) {  // HVD_CFG_LL_PDL: the next launch may be scheduled; memory after the previous grid
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  JtGuard jtg(P.ring.jt);
  constexpr int ESZ = Op::kEsz;
  constexpr int VEL = 16 / ESZ;
  constexpr int HV = VEL / 2;  // elements in half a vector
  constexpr unsigned FULL = 0xffffffffu;
  const RingParams& R = P.ring;
  const RingRank& me = R.rk[blockIdx.y];
  int ch = blockIdx.x;  // -> (buffer b, channel ch of b): a group of buffers may share a launch
  int b = 0;
  while (b + 1 < P.nbuf && ch >= P.bufs[b].nch) ch -= P.bufs[b++].nch;
  const BufDesc& D = P.bufs[b];
  const int nch = D.nch;
  const int N = R.N;
  const int r = me.rank;
  const int T = 2 * (N - 1);
  const unsigned long long flag = ~R.epoch;  // never an LL word nor zeroed memory
  const int par = (int)(R.epoch & 1);
  const unsigned long long qv = D.q / VEL;         // vectors per chunk
  // Lines of 128 B go in pairs: a pair carries 15 vectors (240 B) and two 8 B flags.  In
  // each line lanes 0..6 of an 8-lane group hold 16 B of data; lane 7 holds 8 B of data
  // (half of the pair's vector 7: the low half in the first line, the high half in the
  // second) and the flag.  Wire bytes: 16/15 of the data.
  const unsigned long long pairs = (qv + 14) / 15;
  const unsigned long long slot_words = pairs * 32;  // 2 lines x 16 words per pair
  // the LL128 area follows the two LL halves (the protocols never share memory)
  constexpr unsigned long long kBaseWords = 2 * kLLHalfBytes / 8;
  constexpr unsigned long long kHalfWords = kLL128HalfBytes / 8;
  unsigned long long* const in_ll = me.ll + kBaseWords + (unsigned long long)par * kHalfWords + D.ll_off;
  unsigned long long* const out_ll = me.nll + kBaseWords + (unsigned long long)par * kHalfWords + D.ll_off;
  const unsigned long long ppc = (pairs + nch - 1) / nch;  // pairs of this channel
  const unsigned long long p_lo = (unsigned long long)ch * ppc < pairs ? (unsigned long long)ch * ppc : pairs;
  const unsigned long long p_hi = p_lo + ppc < pairs ? p_lo + ppc : pairs;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, sub = lane % 8, h = (lane >> 3) & 1;
  const unsigned long long nvec = (D.L + VEL - 1) / VEL;
  FusedCtx F = {};
  F.segs = D.segs;
  F.src = D.src + (size_t)blockIdx.y * D.nseg;
  F.dst = D.dst + (size_t)blockIdx.y * D.nseg;
  F.rdst = nullptr;
  F.vbeg = D.vbeg;
  F.tile_seg = D.tile_seg;
  F.tile_vecs = D.tile_vecs;
  F.nseg = D.nseg;
  F.scale_on = P.scale_on;
  F.scale = P.scale;
  F.dtype = P.dtype;
  using Cvt = WireCvt<ESZ, ESZ>;
  SegCache sc;
  bool ok = true;
  unsigned long long sent = 0;
  const bool half = sub == 7;  // this lane carries half of the pair's vector 7
  for (int t = 0; t <= T && ok; ++t) {  // t == T: the chunk received in the last step
    const bool rs = t < N - 1;
    const int s = rs ? t : t - (N - 1);
    const int c = t == T ? mod(r + 2, N) : (rs ? mod(r - s, N) : mod(r + 1 - s, N));
    const unsigned long long c0v = (unsigned long long)c * qv;  // first vector of chunk c
    // a warp moves 2 pairs (4 lines) per step: lanes 0..15 the first pair, 16..31 the second
    for (unsigned long long pg = p_lo + (unsigned long long)warp * 2; pg < p_hi && ok; pg += (blockDim.x / 32) * 2) {
      const unsigned long long pair = pg + lane / 16;
      const bool active = pair < p_hi;
      const unsigned long long line = 2 * pair + h;
      const unsigned long long cvec = pair * 15 + (half ? 7 : sub + 8 * h);  // vector inside the chunk
      const unsigned long long v = c0v + cvec;
      const bool valid = active && cvec < qv && v < nvec;
      unsigned long long left = 0;
      uint4 g = make_uint4(0, 0, 0, 0);
      if (valid) {
        seg_lookup<ESZ>(F, v, sc);
        const unsigned long long e = v * VEL;
        left = sc.end_el > e ? sc.end_el - e : 0;
        if (t <= N - 1 && left) {
          const char* gp = reinterpret_cast<const char*>(sc.g + e * ESZ);
          g = Cvt::fast(gp, left) ? Pack16<ESZ>::conv(__ldcs(reinterpret_cast<const uint4*>(gp)), F.scale, F.scale_on,
                                                      F.dtype)
                                  : Cvt::slow(gp, left, F.scale, F.scale_on, F.dtype);
        }
      }
      if (half && h) g = make_uint4(g.z, g.w, 0, 0);  // the high half of vector 7, in x/y
      uint4 x = g;
      if (t > 0) {
        const unsigned long long* src = in_ll + (unsigned long long)(t - 1) * slot_words + line * 16 + sub * 2;
        bool got = !active;
        unsigned long long a = 0, bw = 0, t0 = 0;
        unsigned spins = 0;
        for (;;) {
          if (!got) asm volatile("ld.relaxed.sys.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(bw) : "l"(src) : "memory");
          const unsigned long long f = __shfl_sync(FULL, bw, (lane & ~7) | 7);
          if (!got && f == flag) got = true;  // the line arrived whole (one 128 B warp store)
          if (__all_sync(FULL, got)) break;
          bool fail = false;
          if ((++spins & 255u) == 0) {
            const unsigned long long now = globaltimer();
            if (t0 == 0) t0 = now;
            else if (now - t0 > R.timeout_ns || *(volatile int*)R.err != 0) fail = true;
          }
          if (__any_sync(FULL, fail)) {
            if (lane == 0) raise_err(R.err, kHvdErrTimeout);
            ok = false;
            break;
          }
        }
        if (!ok) break;
        x = half ? make_uint4((uint32_t)a, (uint32_t)(a >> 32), 0, 0)
                 : make_uint4((uint32_t)a, (uint32_t)(a >> 32), (uint32_t)bw, (uint32_t)(bw >> 32));
        if (t <= N - 1) {
          if (half) Op::template add_words<2>(reinterpret_cast<uint32_t*>(&x), reinterpret_cast<const uint32_t*>(&g));
          else Op::template add_words<4>(reinterpret_cast<uint32_t*>(&x), reinterpret_cast<const uint32_t*>(&g));
        }
      }
      if (t < T && active) {
        unsigned long long* dst = out_ll + (unsigned long long)t * slot_words + line * 16 + sub * 2;
        const unsigned long long w0 = (unsigned long long)x.y << 32 | x.x;
        const unsigned long long w1 = half ? flag : ((unsigned long long)x.w << 32 | x.z);
        asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1,%2};" ::"l"(dst), "l"(w0), "l"(w1) : "memory");
      }
      if (t >= N - 1 && valid && left) {
        char* dp = reinterpret_cast<char*>(sc.d + v * VEL * ESZ);
        if (!half) Cvt::put(dp, left, x);
        else if (left > (unsigned long long)(h * HV)) put_half<ESZ>(dp + h * 8, left - h * HV, x);
      }
    }
    if (t < T) {  // data elements of this channel's pairs of chunk c
      const unsigned long long cl = (unsigned long long)c * D.q;
      unsigned long long ce = cl + D.q < D.L ? cl + D.q : D.L;
      const unsigned long long el = cl + p_lo * 15 * VEL;
      unsigned long long eh = cl + p_hi * 15 * VEL;
      eh = eh < ce ? eh : ce;
      if (eh > el && threadIdx.x == 0) sent += (eh - el) * ESZ;
    }
  }
  if (threadIdx.x == 0) {
    atomicAdd(me.stats + 0, sent);
    if (ch == 0) atomicAdd(me.stats + 1, (unsigned long long)T);
  }
}

// ------------------------------------------------------------------ bulk-copy push ring
// The same ring, chunks, slices, reduction order and signal counters as
// fused_allreduce_kernel, but every byte moves through shared memory by the TMA
// engine's bulk copies (cp.async.bulk) instead of per-thread loads and NVLink
// stores.  Warp roles per CTA (one channel):
//   warp 0  loader      walks the channel's ops, cuts each slice into stages of at
//                       most `stage` bytes, writes a stage descriptor and issues the
//                       bulk loads (gathered gradient pieces -> A, received partial
//                       or forwarded values -> B / A), mbarrier transaction counts;
//                       before the first load of data the predecessor wrote it waits
//                       for the predecessor's counter (acquire, system scope)
//   warps 3+ compute    x = fl32(x * s) (+ partial) in shared memory (the same
//                       per-element operations as the fused kernel: bit-identical),
//                       plus the element-by-element pieces a bulk copy cannot move
//                       (a member's ragged last vector, misaligned tensors)
//   warp 1  storer      issues the stage's bulk stores (successor's scratch / fusion
//                       buffer / tensors over NVLink, own tensors locally), one bulk
//                       group per stage; a stage is retired (its shared memory given
//                       back to the loader, its op published) once its group is
//                       COMPLETE (cp.async.bulk.wait_group)
//   warp 2  signaller   turns the retired op count into the successor's counter with
//                       fence.acq_rel.sys + a relaxed store (the fence is needed:
//                       bulk-group completion alone does not make the writes visible
//                       to the peer, profiles/r02_arrival_probe.json), off the data path
// The storer never waits for the signaller and the loader only for real data
// dependencies, so slices can be small (a fence under load takes ~15 us, which the
// next slices' transfers hide).
constexpr int kBulkComputeWarps = 4;
constexpr int kBulkThreads = (3 + kBulkComputeWarps) * 32;
constexpr int kBulkMaxExc = 16;    // element-wise pieces per stage (the loader cuts the stage when full)
constexpr int kBulkEnd = 15;       // descriptor kind: no more stages
constexpr int kBarCompute = 3;     // named barrier of the compute warps

struct BulkExc {
  unsigned a, n;  // vectors [a, a+n) of the stage (offsets from v0)
  int s, pad;     // member
};
struct StageDesc {
  unsigned long long v0;  // first buffer vector of the stage
  long long pv;           // buffer vector -> channel-private slot shift
  int n;                  // vectors (0: an op without data on this channel)
  int kind;               // FusedKind or kBulkEnd
  int pub;                // ring ops to publish once this stage is complete (-1: none)
  int b;                  // fusion buffer of the call
  int half;               // receive half (scratch / scratch1)
  int nexc;
  int op;                 // op index of this channel (timeline)
  int last;               // last stage of its op
  unsigned long long e_hi;  // end element of the slice (traffic count of a ragged end)
  BulkExc exc[kBulkMaxExc];
};

__host__ __device__ constexpr bool bk_gathers(int k) {
  return k == kF_RS0 || k == kF_RS || k == kF_AG0 || k == kF_RAG0 || k == kF_RAG || k == kF_SOLO;
}
__host__ __device__ constexpr bool bk_scales(int k) {
  return k == kF_RS0 || k == kF_RS || k == kF_AG0 || k == kF_RAG0 || k == kF_SOLO;
}
__host__ __device__ constexpr bool bk_adds(int k) { return k == kF_RS || k == kF_AG0 || k == kF_RAG0; }
__host__ __device__ constexpr bool bk_from_buf(int k) { return k == kF_AG || k == kF_FIN; }
__host__ __device__ constexpr bool bk_to_nscr(int k) { return k == kF_RS0 || k == kF_RS; }
__host__ __device__ constexpr bool bk_to_nbuf(int k) { return k == kF_AG0 || k == kF_AG; }
__host__ __device__ constexpr bool bk_scatters(int k) {
  return k == kF_AG0 || k == kF_AG || k == kF_FIN || k == kF_RAG0 || k == kF_SOLO;
}
__host__ __device__ constexpr bool bk_rscatters(int k) { return k == kF_RAG0 || k == kF_RAG; }
__host__ __device__ constexpr bool bk_members(int k) { return bk_gathers(k) || bk_scatters(k) || bk_rscatters(k); }

__device__ __forceinline__ void mbar_expect_tx_only(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait(int d) {  // until at most d bulk groups are incomplete
  switch (d) {
    case 0: asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.bulk.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.bulk.wait_group 2;" ::: "memory"); break;
    default: asm volatile("cp.async.bulk.wait_group 3;" ::: "memory"); break;
  }
}

// One member's address for this local rank (gather / scatter / successor's scatter).
struct BulkTabs {
  const PackSeg* segs;
  const unsigned long long* vbeg;
  char* const* src;
  char* const* dst;
  char* const* rdst;  // nullptr unless registered
  int nseg;
};
__device__ __forceinline__ BulkTabs bulk_tabs(const FusedParams& P, int b) {
  const BufDesc& D = P.bufs[b];
  BulkTabs T;
  T.segs = D.segs;
  T.vbeg = D.vbeg;
  T.src = D.src + (size_t)blockIdx.y * D.nseg;
  T.dst = D.dst + (size_t)blockIdx.y * D.nseg;
  T.rdst = P.registered ? D.rdst + (size_t)blockIdx.y * D.nseg : nullptr;
  T.nseg = D.nseg;
  return T;
}

// Member of buffer vector v (largest s with vbeg[s] <= v).
__device__ __forceinline__ int bulk_find(const BulkTabs& T, unsigned long long v) {
  int lo = 0, hi = T.nseg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(T.vbeg + mid) <= v) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Walk the members covering buffer vectors [v, vend): f(a, e, s, exc) is called for
// each piece [a, e) of member s; exc: the piece goes element by element (a ragged last
// vector, or a member whose tensor address is not 16 B aligned on this rank).  `s` is
// a cursor (the member of v or one before it).  The loader and the storer make the
// same calls for the same range, so they agree on which pieces are bulk copies.
template <class Fn>
__device__ __forceinline__ void bulk_walk(const BulkTabs& T, int VEL, unsigned long long v, unsigned long long vend,
                                          int& s, Fn&& f) {
  while (s + 1 < T.nseg && __ldg(T.vbeg + s + 1) <= v) ++s;
  while (v < vend && s < T.nseg) {
    const unsigned long long vb = __ldg(T.vbeg + s);
    const unsigned long long cnt = __ldg(&T.segs[s].count);
    const unsigned long long vn = vb + (cnt + VEL - 1) / VEL;  // members are packed on 16 B
    if (vn <= v) {
      ++s;
      continue;
    }
    const unsigned long long e = vend < vn ? vend : vn;
    const uintptr_t al = reinterpret_cast<uintptr_t>(T.src[s]) | reinterpret_cast<uintptr_t>(T.dst[s]) |
                         (T.rdst ? reinterpret_cast<uintptr_t>(T.rdst[s]) : 0);
    const unsigned long long full = vb + cnt / VEL;
    if (al & 15) {
      if (!f(v, e, s, true)) return;
    } else {
      const unsigned long long fe = e < full ? e : full;
      if (fe > v && !f(v, fe, s, false)) return;
      if (e > fe && !f(fe > v ? fe : v, e, s, true)) return;
    }
    v = e;
    if (v >= vn) ++s;
  }
}

// Element-by-element move of one 16 B buffer vector whose member piece cannot be a
// bulk copy: `left` valid elements (the rest of the vector is zero padding).
template <int ESZ>
__device__ __forceinline__ uint4 bulk_gather_elem(const char* p, unsigned long long left) {
  constexpr int VEL = 16 / ESZ;
  alignas(16) unsigned char tmp[16];
#pragma unroll
  for (int i = 0; i < VEL; ++i)
#pragma unroll
    for (int b = 0; b < ESZ; ++b)
      tmp[i * ESZ + b] = (unsigned long long)i < left ? *reinterpret_cast<const volatile unsigned char*>(p + i * ESZ + b) : 0;
  return *reinterpret_cast<const uint4*>(tmp);
}

__device__ __forceinline__ bool mbar_test(unsigned long long* bar, unsigned parity) {
  unsigned done;
  asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return done != 0;
}

// mbarrier wait with the watchdog: a stage that never completes (a protocol bug, a
// peer that died) latches HVD_ERR_TIMEOUT and traps instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait_wd(unsigned long long* bar, unsigned parity, int* err,
                                             unsigned long long timeout_ns) {
  unsigned done = 0, spins = 0;
  unsigned long long t0 = 0;
  for (;;) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    if (done) return;
    if ((++spins & 255u) == 0) {
      const unsigned long long now = globaltimer();
      if (t0 == 0) {
        t0 = now;
      } else if (now - t0 > timeout_ns + 1000000000ull) {  // after the spin watchdogs had their chance
        raise_err(err, kHvdErrTimeout);
        __threadfence_system();
        asm volatile("trap;");
      }
    }
  }
}

template <class Op>
__global__ void __launch_bounds__(kBulkThreads, 1) bulk_allreduce_kernel(const __grid_constant__ FusedParams P) {
  JtGuard jtg(P.ring.jt);
  extern __shared__ __align__(1024) unsigned char s_bulk[];
  constexpr int ESZ = Op::kEsz;
  constexpr int VEL = 16 / ESZ;
  const RingParams& R = P.ring;
  const RingRank& me = R.rk[blockIdx.y];
  const int ch = blockIdx.x;
  const int N = R.N;
  const int r = me.rank;
  const int T = 2 * (N - 1);
  const int S = P.bulk_stages;
  const unsigned stage_vecs = (unsigned)(P.bulk_stage_bytes / 16);
  const unsigned long long base0 = R.base[ch];
  // shared memory: [A stages][B stages (N > 1)][descriptors][mbarriers full, comp, empty]
  uint4* sA = reinterpret_cast<uint4*>(s_bulk);
  uint4* sB = sA + (size_t)S * stage_vecs;
  StageDesc* desc = reinterpret_cast<StageDesc*>(sA + (size_t)(N > 1 ? 2 : 1) * S * stage_vecs);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(desc + S);
  unsigned long long* comp = full + S;
  unsigned long long* empty = comp + S;
  __shared__ int s_abort, s_done;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    s_abort = 0;
    s_done = 0;
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&comp[i], kBulkComputeWarps);
      mbar_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // programmatic dependent launch (N = 1 launches): the next kernel on the stream may
    // start launching now; it waits for this grid's completion before touching memory
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  __syncthreads();
  // ring ops this channel publishes over the whole call
  int total = 0;
  for (int b = 0; b < P.nbuf; ++b)
    if (chan_of(P.bufs[b], ch, gridDim.x) >= 0) total += T * P.bufs[b].K;

  if (warp == 2) {  // ---- signaller: handshake to the predecessor, then publish retired ops
    if (lane == 0) {
      st_relaxed_sys(me.phash + ch, R.hash);
      st_release_sys(me.pready + ch, R.epoch);
      if (total > 0)
        signal_loop(&s_done, total, me.nflags + ch, base0, R.sig_mode, nullptr,
                    R.tl ? R.tl + tl_words(R.tl_max) * blockIdx.y + ((size_t)kMaxChannels + ch) * R.tl_max * 2 : nullptr,
                    R.tl_max);
    }
    return;
  }
  unsigned long long* tl_d = R.tl ? R.tl + tl_words(R.tl_max) * blockIdx.y + (size_t)ch * R.tl_max * 2 : nullptr;

  if (warp == 0) {  // ---- loader
    if (lane != 0) return;
    unsigned long long seq = 0;
    unsigned long long bbase = base0;
    int ring_i = 0, bpar = 0, nop = 0;
    bool abort = false;
    auto acquire_slot = [&](unsigned long long q) -> int {
      const int slot = (int)(q % S);
      if (q >= (unsigned long long)S) mbar_wait_wd(&empty[slot], (unsigned)((q / S - 1) & 1), R.err, R.timeout_ns);
      return slot;
    };
    // member pieces of stage [v0, v1): bulk-load the gathered ones into A, list the
    // element-wise ones; the stage ends early (returned end) when the list is full
    auto walk_stage = [&](StageDesc& sd, int slot, unsigned long long v0, unsigned long long v1, int kind,
                          const BulkTabs& TB, int& cur) -> unsigned long long {
      uint4* A = sA + (size_t)slot * stage_vecs;
      unsigned long long cut = v1;
      int nexc = 0;
      bulk_walk(TB, VEL, v0, v1, cur, [&](unsigned long long a, unsigned long long e, int s, bool exc) -> bool {
        if (exc) {
          if (nexc == kBulkMaxExc) {
            cut = a;
            return false;
          }
          sd.exc[nexc].a = (unsigned)(a - v0);
          sd.exc[nexc].n = (unsigned)(e - a);
          sd.exc[nexc].s = s;
          ++nexc;
        } else if (bk_gathers(kind) && !abort) {
          const unsigned bytes = (unsigned)((e - a) * 16);
          mbar_expect_tx_only(&full[slot], bytes);
          tma_load(A + (a - v0), TB.src[s] + (a - __ldg(TB.vbeg + s)) * 16, bytes, &full[slot]);
        }
        return true;
      });
      sd.nexc = nexc;
      return cut;
    };
    if (N == 1) {  // no ring: tiles of `stage` bytes round robin over the channels
      asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous grid on the stream is complete
      for (int b = 0; b < P.nbuf; ++b) {
        const BufDesc& D = P.bufs[b];
        const BulkTabs TB = bulk_tabs(P, b);
        const unsigned long long nvec = (D.L + VEL - 1) / VEL;
        for (unsigned long long vlo = (unsigned long long)ch * stage_vecs; vlo < nvec;
             vlo += (unsigned long long)gridDim.x * stage_vecs) {
          const unsigned long long vhi = vlo + stage_vecs < nvec ? vlo + stage_vecs : nvec;
          int cur = bulk_find(TB, vlo);
          for (unsigned long long v0 = vlo; v0 < vhi;) {
            const int slot = acquire_slot(seq);
            StageDesc& sd = desc[slot];
            const unsigned long long v1 = walk_stage(sd, slot, v0, vhi, kF_SOLO, TB, cur);
            sd.v0 = v0;
            sd.pv = 0;
            sd.n = (int)(v1 - v0);
            sd.kind = kF_SOLO;
            sd.pub = -1;
            sd.b = b;
            sd.half = 0;
            sd.op = 0;
            sd.last = 0;
            sd.e_hi = D.L;
            mbar_arrive(&full[slot]);
            ++seq;
            v0 = v1;
          }
        }
      }
      const int slot = acquire_slot(seq);
      desc[slot].kind = kBulkEnd;
      mbar_arrive(&full[slot]);
      return;
    }
    for (int b = 0; b < P.nbuf; ++b) {
      const BufDesc& D = P.bufs[b];
      const int cg = chan_of(D, ch, gridDim.x);
      if (cg < 0) continue;
      const int K = D.K;
      const int half = bpar;
      bpar ^= 1;
      const BulkTabs TB = bulk_tabs(P, b);
      const char* scr = half ? me.scratch1 : me.scratch;
      const int nops = P.registered ? T * K : (T + 1) * K;
      int cur = 0;  // member cursor (ranges grow within a slice)
      for (int j = 0; j < nops; ++j, ++nop) {
        int t, k;
        if (P.registered) {
          t = j / K;
          k = j - t * K;
        } else {
          fused_op(j, K, T, R.fin_lag, t, k);
        }
        const bool rs = t < N - 1;
        const int s_ = rs ? t : t - (N - 1);
        const int c = t == T ? mod(r + 2, N) : (rs ? mod(r - s_, N) : mod(r + 1 - s_, N));
        int kind;
        if (P.registered) kind = t == 0 ? kF_RS0 : (rs ? kF_RS : (s_ == 0 ? kF_RAG0 : kF_RAG));
        else kind = t == T ? kF_FIN : (t == 0 ? kF_RS0 : (rs ? kF_RS : (s_ == 0 ? kF_AG0 : kF_AG)));
        unsigned long long lo, hi;
        slice_range_d(D, c, cg, k, lo, hi);
        const long long pv =
            (long long)(((unsigned long long)ch * P.region_el + (unsigned long long)c * D.ch_el +
                         (lo - (unsigned long long)c * D.q - (unsigned long long)cg * D.ch_el)) / VEL) -
            (long long)(lo / VEL);
        const unsigned long long vlo = lo / VEL, vhi = hi > lo ? (hi + VEL - 1) / VEL : vlo;
        const int pub = t < T ? ++ring_i : -1;
        const unsigned long long target = t > 0 ? bbase + (unsigned long long)(t - 1) * K + k + 1 : 0;
        if (tl_d && nop < R.tl_max) tl_d[2 * nop] = globaltimer();
        bool dep_done = target == 0;
        auto wait_dep = [&]() {
          if (dep_done) return;
          dep_done = true;
          if (!abort && !spin_until(me.flags + ch, target, R.err, R.timeout_ns)) {
            abort = true;
            s_abort = 1;
#ifdef HVD_BULK_DEBUG
            printf("bulk dep timeout r=%d ch=%d kind=%d t=%d k=%d target=%llu have=%llu base0=%llu\n", r, ch, kind, t, k,
                   target, *(volatile unsigned long long*)(me.flags + ch), base0);
#endif
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");  // the acquire covers the async-proxy loads
        };
        if (vhi <= vlo) {  // no data on this channel: an empty stage keeps the publish order
          const int slot = acquire_slot(seq);
          StageDesc& sd = desc[slot];
          sd.v0 = vlo;
          sd.pv = pv;
          sd.n = 0;
          sd.kind = kind;
          sd.pub = pub;
          sd.b = b;
          sd.half = half;
          sd.nexc = 0;
          sd.op = nop;
          sd.last = 1;
          sd.e_hi = hi;
          mbar_arrive(&full[slot]);
          ++seq;
          continue;
        }
        cur = bk_members(kind) ? bulk_find(TB, vlo) : 0;
        for (unsigned long long v0 = vlo; v0 < vhi;) {
          const int slot = acquire_slot(seq);
          StageDesc& sd = desc[slot];
          uint4* A = sA + (size_t)slot * stage_vecs;
          uint4* B = sB + (size_t)slot * stage_vecs;
          unsigned long long v1 = v0 + stage_vecs < vhi ? v0 + stage_vecs : vhi;
          const bool dep_gather = kind == kF_RAG;  // own tensors written by the predecessor
          if (dep_gather) wait_dep();
          sd.nexc = 0;
          if (bk_members(kind)) v1 = walk_stage(sd, slot, v0, v1, kind, TB, cur);
          const int nexc = sd.nexc;
          if (bk_adds(kind) || bk_from_buf(kind)) {
            wait_dep();
            if (!abort) {
              const unsigned bytes = (unsigned)((v1 - v0) * 16);
              mbar_expect_tx_only(&full[slot], bytes);
              if (bk_adds(kind)) tma_load(B, scr + (v0 + pv) * 16, bytes, &full[slot]);
              else tma_load(A, me.buf + (v0 + pv) * 16, bytes, &full[slot]);
            }
          }
          sd.v0 = v0;
          sd.pv = pv;
          sd.n = (int)(v1 - v0);
          sd.kind = kind;
          sd.pub = v1 >= vhi ? pub : -1;
          sd.b = b;
          sd.half = half;
          sd.op = nop;
          sd.last = v1 >= vhi;
          sd.e_hi = hi;
          if (nexc) wait_dep();  // element-wise gathers of RAG data by the compute warps
          mbar_arrive(&full[slot]);
          ++seq;
          v0 = v1;
        }
      }
      bbase += (unsigned long long)T * K;
    }
    const int slot = acquire_slot(seq);
    desc[slot].kind = kBulkEnd;
    mbar_arrive(&full[slot]);
    // registered: the predecessor's last all-gather stores land in this rank's tensors;
    // the kernel completes only when they have arrived
    if (P.registered && total > 0 && !abort) spin_until(me.flags + ch, bbase, R.err, R.timeout_ns);
    return;
  }

  if (warp == 1) {  // ---- storer
    if (lane != 0) return;
    unsigned long long seq = 0, retired = 0;
    unsigned long long sent = 0;
    bool ready = false;
    const int depth = P.bulk_depth;
    // A stage's shared memory goes back to the loader as soon as its bulk stores have READ
    // it (cp.async.bulk.wait_group.read); its op is published once the stores are COMPLETE
    // (cp.async.bulk.wait_group), `depth` groups behind the newest.  The publish data of
    // a stage is kept here because its descriptor slot is reused after the release.
    constexpr int kRing = 8;
    int r_pub[kRing], r_op[kRing];
    bool r_last[kRing];
    unsigned long long released = 0;
    auto release = [&](unsigned long long upto) {  // stages < upto have been read
      for (; released < upto; ++released) mbar_arrive(&empty[(int)(released % S)]);
    };
    auto retire = [&](unsigned long long upto) {  // stages < upto are complete
      release(upto);
      for (; retired < upto; ++retired) {
        const int i = (int)(retired % kRing);
        if (r_pub[i] >= 0) st_release_cta_shared(&s_done, r_pub[i]);
        if (r_last[i] && tl_d && r_op[i] < R.tl_max) tl_d[2 * r_op[i] + 1] = globaltimer();
      }
    };
    for (;; ++seq) {
      const int slot = (int)(seq % S);
      // the next stage may wait on the successor's progress, which may wait on a stage
      // published here: never leave issued stages unpublished while waiting for it
      if (N > 1 && retired < seq && !mbar_test(&comp[slot], (unsigned)((seq / S) & 1))) {
        bulk_wait(0);
        retire(seq);
      }
      mbar_wait_wd(&comp[slot], (unsigned)((seq / S) & 1), R.err, R.timeout_ns);
      const StageDesc& sd = desc[slot];
      const int kind = sd.kind;
      if (kind == kBulkEnd) break;
      const uint4* A = sA + (size_t)slot * stage_vecs;
      if (sd.n > 0 && !s_abort) {
        const bool remote = bk_to_nscr(kind) || bk_to_nbuf(kind) || bk_rscatters(kind);
        if (remote && !ready) {  // the launch's first remote store waits for the successor
          ready = true;
          if (!spin_until(me.rflags + ch, R.epoch, R.err, R.timeout_ns)) {
            s_abort = 1;
#ifdef HVD_BULK_DEBUG
            printf("bulk handshake timeout r=%d ch=%d epoch=%llu have=%llu\n", r, ch, R.epoch,
                   *(volatile unsigned long long*)(me.rflags + ch));
#endif
          } else if (*(volatile const unsigned long long*)(me.rhash + ch) != R.hash) {
            raise_err(R.err, kHvdErrMismatch);
            s_abort = 1;
          }
        }
        if (!s_abort) {
          const unsigned bytes = (unsigned)sd.n * 16;
          if (bk_to_nscr(kind)) bulk_store((sd.half ? me.nscratch1 : me.nscratch) + (sd.v0 + sd.pv) * 16, A, bytes);
          if (bk_to_nbuf(kind)) bulk_store(me.nbuf + (sd.v0 + sd.pv) * 16, A, bytes);
          if (remote) {
            const unsigned long long eh = (sd.v0 + sd.n) * VEL < sd.e_hi ? (sd.v0 + sd.n) * VEL : sd.e_hi;
            sent += (eh - sd.v0 * VEL) * ESZ;
          }
          if (bk_scatters(kind) || bk_rscatters(kind)) {
            const BulkTabs TB = bulk_tabs(P, sd.b);
            int cur = bulk_find(TB, sd.v0);
            bulk_walk(TB, VEL, sd.v0, sd.v0 + sd.n, cur,
                      [&](unsigned long long a, unsigned long long e, int s, bool exc) -> bool {
                        if (!exc) {
                          const unsigned long long off = (a - __ldg(TB.vbeg + s)) * 16;
                          if (bk_scatters(kind)) bulk_store(TB.dst[s] + off, A + (a - sd.v0), (unsigned)((e - a) * 16));
                          if (bk_rscatters(kind)) bulk_store(TB.rdst[s] + off, A + (a - sd.v0), (unsigned)((e - a) * 16));
                        }
                        return true;
                      });
          }
        }
      }
      bulk_commit();
      r_pub[seq % kRing] = sd.pub;
      r_op[seq % kRing] = sd.op;
      r_last[seq % kRing] = sd.last != 0;
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      if (seq > 0) release(seq);  // all but the newest stage have been read
      if (N == 1) continue;       // nothing to publish: the stores complete with the grid
      bulk_wait(depth);
      if (seq + 1 > (unsigned long long)depth) retire(seq + 1 - depth);
    }
    bulk_wait(0);
    retire(seq);
    atomicAdd(me.stats + 0, sent);
    if (ch == 0) atomicAdd(me.stats + 1, (unsigned long long)T * P.nbuf);
    return;
  }

  // ---- compute warps
  const int ctid = threadIdx.x - 96;
  constexpr int CT = kBulkComputeWarps * 32;
  const float scale = P.scale;
  const int scale_on = P.scale_on;
  for (unsigned long long seq = 0;; ++seq) {
    const int slot = (int)(seq % S);
    mbar_wait_wd(&full[slot], (unsigned)((seq / S) & 1), R.err, R.timeout_ns);
    const StageDesc& sd = desc[slot];
    const int kind = sd.kind;
    if (kind == kBulkEnd) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&comp[slot]);
      break;
    }
    uint4* A = sA + (size_t)slot * stage_vecs;
    const uint4* B = sB + (size_t)slot * stage_vecs;
    const int n = sd.n;
    const int nexc = sd.nexc;
    if (nexc && bk_gathers(kind)) {
      const BulkTabs TB = bulk_tabs(P, sd.b);
      for (int x = 0; x < nexc; ++x) {
        const BulkExc ex = sd.exc[x];
        const unsigned long long dst_off = TB.segs[ex.s].dst_off;
        const unsigned long long end_el = dst_off + TB.segs[ex.s].count;
        for (unsigned i = ctid; i < ex.n; i += CT) {
          const unsigned long long e = (sd.v0 + ex.a + i) * VEL;
          A[ex.a + i] = bulk_gather_elem<ESZ>(TB.src[ex.s] + (e - dst_off) * ESZ, end_el - e);
        }
      }
      bar_sync(kBarCompute, CT);
    }
    if (bk_scales(kind) || bk_adds(kind)) {
      const int on = bk_scales(kind) ? scale_on : 0;
      for (int v = ctid; v < n; v += CT) {
        uint4 x = A[v];
        if (on) x = Pack16<ESZ>::conv(x, scale, 1, P.dtype);
        if (bk_adds(kind)) {
          const uint4 y = B[v];
          Op::template add_words<4>(reinterpret_cast<uint32_t*>(&x), reinterpret_cast<const uint32_t*>(&y));
        }
        A[v] = x;
      }
    }
    if (nexc && (bk_scatters(kind) || bk_rscatters(kind))) {
      bar_sync(kBarCompute, CT);
      const BulkTabs TB = bulk_tabs(P, sd.b);
      for (int x = 0; x < nexc; ++x) {
        const BulkExc ex = sd.exc[x];
        const unsigned long long dst_off = TB.segs[ex.s].dst_off;
        const unsigned long long end_el = dst_off + TB.segs[ex.s].count;
        for (unsigned i = ctid; i < ex.n; i += CT) {
          const unsigned long long e = (sd.v0 + ex.a + i) * VEL;
          const uint4 val = A[ex.a + i];
          if (bk_scatters(kind)) scatter_slow<ESZ>(TB.dst[ex.s] + (e - dst_off) * ESZ, end_el - e, val);
          if (bk_rscatters(kind)) scatter_slow<ESZ>(TB.rdst[ex.s] + (e - dst_off) * ESZ, end_el - e, val);
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> bulk-store reads
    __syncwarp();
    if (lane == 0) mbar_arrive(&comp[slot]);
  }
}


// ------------------------------------------------------------------ LL128 line-atomicity self-test
// hvd_ll128_selftest / hvd_connect: LL128 relies on a warp's 128-byte line store arriving
// whole, which PTX does not promise.  Every rank writes `rounds` x (gridDim.x x
// lines_per_cta) lines into its successor's LL128 area (half 0) — lanes 0..6 of an
// 8-lane group a pattern of (round, line, lane), lane 7 the flag ~(tag + round), one warp
// store per line, exactly as ll128_allreduce_kernel stores — while its other warps read
// the lines its predecessor writes into its own area.  A line whose flag matches but
// whose data does not is torn; the count goes to `torn`.  Lines that never arrive within
// the watchdog count as well.  The tag keeps the flags far from any LL128 epoch.
constexpr unsigned long long kSelfTestTag = 0x5e1f000000000000ull;

__device__ __forceinline__ unsigned long long selftest_word(int round, unsigned long long line, int sub, int half) {
  unsigned long long z = kSelfTestTag ^ ((unsigned long long)round << 40) ^ (line << 8) ^ ((unsigned long long)sub << 1) ^
                         (unsigned long long)half;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void __launch_bounds__(256) ll128_selftest_kernel(const __grid_constant__ RingParams P, int rounds,
                                                             int lines_per_cta, unsigned long long* torn) {
  constexpr unsigned FULL = 0xffffffffu;
  const RingRank& me = P.rk[blockIdx.y];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, sub = lane % 8, grp = lane / 8;
  constexpr unsigned long long kBaseWords = 2 * kLLHalfBytes / 8;  // LL128 half 0
  const unsigned long long* in = me.ll + kBaseWords;
  unsigned long long* out = me.nll + kBaseWords;
  const unsigned long long lines_total = (unsigned long long)gridDim.x * lines_per_cta;
  const unsigned long long l0 = (unsigned long long)blockIdx.x * lines_per_cta;
  const int w = warp & 3;
  // handshake: this rank's earlier launches are over (the host synchronised the device),
  // so its LL128 area may be overwritten; the writers wait for the successor's word
  if (threadIdx.x == 0) st_release_sys(me.pready + blockIdx.x, P.epoch);
  if (warp < 4) {  // writers: the successor's area
    if (lane == 0) spin_until(me.rflags + blockIdx.x, P.epoch, P.err, P.timeout_ns);  // a dead peer latches TIMEOUT
    __syncwarp();
    for (int r = 0; r < rounds; ++r)
      for (unsigned long long l = l0 + w * 4 + grp; l < l0 + lines_per_cta; l += 16) {
        unsigned long long* dst = out + ((unsigned long long)r * lines_total + l) * 16 + sub * 2;
        const unsigned long long f = ~(kSelfTestTag + (unsigned long long)r);
        const unsigned long long w0 = sub < 7 ? selftest_word(r, l, sub, 0) : f;
        const unsigned long long w1 = sub < 7 ? selftest_word(r, l, sub, 1) : f;
        asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1,%2};" ::"l"(dst), "l"(w0), "l"(w1) : "memory");
      }
    return;
  }
  // readers: poll this rank's area, line by line, and check every arrived line
  unsigned long long bad = 0;
  bool dead = false;
  for (int r = 0; r < rounds && !dead; ++r) {
    const unsigned long long f = ~(kSelfTestTag + (unsigned long long)r);
    for (unsigned long long lg = l0 + w * 4; lg < l0 + lines_per_cta && !dead; lg += 16) {
      const unsigned long long l = lg + grp;
      const bool active = l < l0 + lines_per_cta;
      const unsigned long long* src = in + ((unsigned long long)r * lines_total + l) * 16 + sub * 2;
      unsigned long long a = 0, b = 0, t0 = 0;
      bool got = !active;
      unsigned spins = 0;
      for (;;) {
        if (!got) asm volatile("ld.relaxed.sys.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(src) : "memory");
        const unsigned long long fl = __shfl_sync(FULL, b, (lane & ~7) | 7);
        if (!got && fl == f) got = true;
        if (__all_sync(FULL, got)) break;
        bool fail = false;
        if ((++spins & 255u) == 0) {
          const unsigned long long now = globaltimer();
          if (t0 == 0) t0 = now;
          else if (now - t0 > P.timeout_ns) fail = true;
        }
        if (__any_sync(FULL, fail)) {
          dead = true;
          break;
        }
      }
      if (dead) break;
      const bool ok = !active || (sub < 7 ? (a == selftest_word(r, l, sub, 0) && b == selftest_word(r, l, sub, 1))
                                          : (a == f && b == f));
      const unsigned ballot = __ballot_sync(FULL, !ok);
      if (lane == 0) bad += (unsigned long long)__popc(ballot);
    }
  }
  if (lane == 0) {
    if (dead) bad += 1ull << 32;  // lines that never arrived
    if (bad) atomicAdd(torn + blockIdx.y, bad);
  }
}

struct BufList { char* b[kMaxLocal]; };

template <int ESZ>
__global__ void __launch_bounds__(512) scale_kernel(const BufList bufs, unsigned long long count, float s,
                                                    int dtype, const JtRef jt) {
  JtGuard jtg(jt);
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
constexpr int kMaxDevices = 64;

// Kernels actually launched (a launcher with no work returns without one): the host
// counts launches and opens timeline records only for launches that happened.
static unsigned long long g_launched = 0;
unsigned long long kernels_launched() { return g_launched; }
template <bool PACK>
static cudaError_t launch_pack_impl(const PackParams& p, int dtype, int nlocal, int grid, int threads,
                                    cudaStream_t s) {
  if (p.ntiles == 0) return cudaSuccess;
  unsigned long long g = p.ntiles < (unsigned long long)grid ? p.ntiles : (unsigned long long)grid;
  dim3 gd((unsigned)g, nlocal);
  ++g_launched;
  switch (elem_size(dtype)) {
    case 4: pack_kernel<4, PACK><<<gd, threads, 0, s>>>(p, dtype); break;
    case 2: pack_kernel<2, PACK><<<gd, threads, 0, s>>>(p, dtype); break;
    case 8: pack_kernel<8, PACK><<<gd, threads, 0, s>>>(p, dtype); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_jt_clock(unsigned long long* host_out, cudaStream_t s) {
  jt_clock_kernel<<<1, 1, 0, s>>>(host_out);
  return cudaGetLastError();
}

cudaError_t launch_pack(const PackParams& p, int dtype, int nlocal, int grid, int threads, cudaStream_t s) {
  return launch_pack_impl<true>(p, dtype, nlocal, grid, threads, s);
}

cudaError_t launch_unpack(const PackParams& p, int dtype, int nlocal, int grid, int threads, cudaStream_t s) {
  return launch_pack_impl<false>(p, dtype, nlocal, grid, threads, s);
}

cudaError_t launch_scale(char* const* bufs, int nlocal, unsigned long long count, int dtype, float scale,
                         int grid, int threads, const JtRef& jt, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  BufList b = {};
  for (int i = 0; i < nlocal && i < kMaxLocal; ++i) b.b[i] = bufs[i];
  dim3 gd(grid, nlocal);
  ++g_launched;
  switch (elem_size(dtype)) {
    case 4: scale_kernel<4><<<gd, threads, 0, s>>>(b, count, scale, dtype, jt); break;
    case 2: scale_kernel<2><<<gd, threads, 0, s>>>(b, count, scale, dtype, jt); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <class Op>
static cudaError_t launch_ring_t(const RingParams& p, int nch, int nlocal, int threads, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nch, nlocal);
  cfg.blockDim = dim3(threads + 32);  // + signal warp
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (they wait on each other)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ++g_launched;
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

// N == 1: the whole allreduce is gather x (1/N) -> scatter of every member
// (plus the wire round trip, R14).  A plain HBM stream: no ring, no signals,
// so none of the fused kernel's machinery.  One CTA per tile of kSoloThreads x U
// wire vectors over all buffers of the call (the block scheduler balances the
// tail; a persistent grid-stride walk left the SMs idle 28 % of the kernel in
// ncu).  A tile inside one member with aligned addresses (the common case)
// issues its U independent 16 B loads off one pointer, then its U stores.
#ifndef HVD_SOLO_TMA
#define HVD_SOLO_TMA 1
#endif
constexpr int kSoloThreads = HVD_SOLO_THREADS;
constexpr int kSoloU = HVD_SOLO_U;  // 16 B wire vectors per thread (same-dtype wire)
constexpr int kSoloSegCache = 256;  // member starts a boundary tile stages in shared memory

// A member's partial last vector (fewer than 16 / ESZ elements), same dtype.
template <int ESZ>
__device__ __noinline__ void solo_ragged(char* d, const char* g, unsigned left, float scale, int on, int dtype) {
  scatter_slow<ESZ>(d, left, Pack16<ESZ>::conv(gather_slow<ESZ>(g, left), scale, on, dtype));
}

#ifndef HVD_SOLO_MINB
#define HVD_SOLO_MINB 0  // > 0: CTAs per SM the register allocation must allow
#endif
#if HVD_SOLO_MINB
#define HVD_SOLO_BOUNDS __launch_bounds__(kSoloThreads, HVD_SOLO_MINB)
#else
#define HVD_SOLO_BOUNDS __launch_bounds__(kSoloThreads)
#endif
template <class Op, int TESZ>
__global__ void HVD_SOLO_BOUNDS solo_kernel(const __grid_constant__ FusedParams P) {
  JtGuard jtg(P.ring.jt);
  constexpr int ESZ = Op::kEsz;
  constexpr int VEL = 16 / ESZ;
  constexpr int U = TESZ > ESZ ? (kSoloU + 1) / 2 : kSoloU;  // fp32 tensor, bf16 wire: 32 B of tensor each
  constexpr unsigned long long TILE = (unsigned long long)kSoloThreads * U;
  using Cvt = WireCvt<ESZ, TESZ>;
  const unsigned tid = threadIdx.x;
  // same dtype: the tile's bulk-copy staging (one per CTA, shared by every tile path)
  __shared__ __align__(128) uint4 s_tile[TESZ == ESZ ? TILE * kSoloTPC : 1];
  __shared__ __align__(8) unsigned long long s_bar;
  // programmatic dependent launch: the next kernel on the stream may be launched as soon
  // as every CTA of this grid has started; this grid's own memory work waits for the
  // previous grid's completion (griddepcontrol.wait), so back-to-back calls overlap only
  // the launch, never the data.  Member-tile descriptors are plan tables no kernel writes:
  // they are read before the wait.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#if HVD_SOLO_TMA
  if constexpr (TESZ == ESZ && kSoloTPC > 1) {
    if (P.solo_tpc > 1) {
      // several member tiles per CTA (every tile of the launch a plain bulk copy): all
      // descriptors in one round trip, all bulk loads in flight, each store as its load lands
      __shared__ __align__(8) unsigned long long s_bars[kSoloTPC];
      uint4 dA[kSoloTPC], dB[kSoloTPC];
      bool ok[kSoloTPC];
#pragma unroll
      for (int j = 0; j < kSoloTPC; ++j) {
        unsigned long long tj = (unsigned long long)blockIdx.x * kSoloTPC + j;
        int bj = 0;
        for (; bj < P.nbuf; ++bj) {
          if (tj < P.bufs[bj].nstile) break;
          tj -= P.bufs[bj].nstile;
        }
        ok[j] = bj < P.nbuf;
        if (ok[j]) {
          const uint4* q = reinterpret_cast<const uint4*>(P.bufs[bj].stile + tj);
          dA[j] = __ldg(q);
          dB[j] = __ldg(q + 1);
        }
      }
      asm volatile("griddepcontrol.wait;" ::: "memory");
      if (tid == 0) {
#pragma unroll
        for (int j = 0; j < kSoloTPC; ++j)
          if (ok[j] && dB[j].x) {
            mbar_init(&s_bars[j], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            mbar_expect_tx(&s_bars[j], dB[j].x);
            tma_load(s_tile + j * TILE, reinterpret_cast<const char*>((unsigned long long)dA[j].x | ((unsigned long long)dA[j].y << 32)),
                     dB[j].x, &s_bars[j]);
          }
#pragma unroll
        for (int j = 0; j < kSoloTPC; ++j)
          if (ok[j] && dB[j].x) {
            mbar_wait(&s_bars[j], 0);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         ::"l"((unsigned long long)dA[j].z | ((unsigned long long)dA[j].w << 32)),
                         "r"(smem_u32(s_tile + j * TILE)), "r"(dB[j].x) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      } else if (tid == 32) {
#pragma unroll
        for (int j = 0; j < kSoloTPC; ++j)
          if (ok[j] && dB[j].y) {
            const char* g = reinterpret_cast<const char*>((unsigned long long)dA[j].x | ((unsigned long long)dA[j].y << 32));
            char* d = reinterpret_cast<char*>((unsigned long long)dA[j].z | ((unsigned long long)dA[j].w << 32));
            solo_ragged<ESZ>(d + dB[j].x, g + dB[j].x, dB[j].y, P.scale, P.scale_on, P.dtype);
          }
      }
      return;
    }
  }
#endif
  unsigned long long t = blockIdx.x;  // -> (buffer b, tile t of b)
  int b = 0;
  for (; b < P.nbuf; ++b) {
    const unsigned long long nt =
        P.bufs[b].stile ? P.bufs[b].nstile : ((P.bufs[b].L + VEL - 1) / VEL + TILE - 1) / TILE;
    if (t < nt) break;
    t -= nt;
  }
  if (b == P.nbuf) return;
  const BufDesc& D = P.bufs[b];
#if HVD_SOLO_TMA
  if constexpr (TESZ == ESZ) {
    if (D.stile) {
      // member tile (built with the plan): one descriptor load, then bulk copies
      const uint4* dp4 = reinterpret_cast<const uint4*>(D.stile + t);
      const uint4 d0v = __ldg(dp4), d1v = __ldg(dp4 + 1);
      asm volatile("griddepcontrol.wait;" ::: "memory");
      const char* gsrc = reinterpret_cast<const char*>((unsigned long long)d0v.x | ((unsigned long long)d0v.y << 32));
      char* gdst = reinterpret_cast<char*>((unsigned long long)d0v.z | ((unsigned long long)d0v.w << 32));
      const unsigned bytes = d1v.x, ragged = d1v.y;
      if (!(d1v.z & 1u)) {
        if (bytes) {
          if (tid == 0) {
            mbar_init(&s_bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            mbar_expect_tx(&s_bar, bytes);
            tma_load(s_tile, gsrc, bytes, &s_bar);
          }
          if (ragged && tid == 32)  // the member's partial last vector, element by element
            solo_ragged<ESZ>(gdst + bytes, gsrc + bytes, ragged, P.scale, P.scale_on, P.dtype);
          __syncthreads();
          if (P.scale_on) {
            mbar_wait(&s_bar, 0);
            for (unsigned v = tid; v < bytes / 16; v += kSoloThreads)
              s_tile[v] = Pack16<ESZ>::conv(s_tile[v], P.scale, P.scale_on, P.dtype);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
          } else if (tid == 0) {
            mbar_wait(&s_bar, 0);
          }
          if (tid == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         ::"l"(gdst), "r"(smem_u32(s_tile)), "r"(bytes) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
        } else if (ragged && tid == 0) {
          solo_ragged<ESZ>(gdst, gsrc, ragged, P.scale, P.scale_on, P.dtype);
        }
        return;
      }
    }
  }
#endif
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (a no-op after the wait above)
  FusedCtx F = {};
  F.segs = D.segs;
  F.src = D.src + (size_t)blockIdx.y * D.nseg;
  F.dst = D.dst + (size_t)blockIdx.y * D.nseg;
  F.rdst = nullptr;
  F.vbeg = D.vbeg;
  F.tile_seg = D.tile_seg;
  F.tile_vecs = D.tile_vecs;
  F.nseg = D.nseg;
  F.scale_on = P.scale_on;
  F.scale = P.scale;
  F.dtype = P.dtype;
  SegCache sc;
  const unsigned long long nvec = (D.L + VEL - 1) / VEL;
  unsigned long long base = t * TILE;
  unsigned long long t_end = base + TILE < nvec ? base + TILE : nvec;
  if (D.stile) {  // a misaligned member's tile: buffer vectors [src, dst) of the descriptor
    base = D.stile[t].src;
    t_end = D.stile[t].dst;
  }
  seg_lookup<TESZ>(F, base, sc);
  const unsigned long long e0 = base * VEL;
  const char* g0 = reinterpret_cast<const char*>(sc.g + e0 * TESZ);
  char* d0 = reinterpret_cast<char*>(sc.d + e0 * TESZ);
  const bool fast = t_end * VEL <= sc.end_el && t_end <= sc.vhi &&
                    ((reinterpret_cast<uintptr_t>(g0) | reinterpret_cast<uintptr_t>(d0)) & 15) == 0;
#if HVD_SOLO_TMA
  if constexpr (TESZ == ESZ) {
    // same dtype: the tile moves HBM -> shared -> HBM by bulk copies (TMA engine), the
    // threads only scale it in shared memory; in-flight bytes cost shared memory, not
    // registers (~14 CTAs x 16 KiB per SM)
    if (fast) {
      const unsigned bytes = (unsigned)((t_end - base) * 16);
      if (tid == 0) {
        mbar_init(&s_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_expect_tx(&s_bar, bytes);
        tma_load(s_tile, g0, bytes, &s_bar);
      }
      __syncthreads();
      if (F.scale_on) {  // (N = 1 sums and averages by 1 move the tile unchanged)
        mbar_wait(&s_bar, 0);
        for (unsigned long long v = tid; v < t_end - base; v += kSoloThreads)
          s_tile[v] = Pack16<ESZ>::conv(s_tile[v], F.scale, F.scale_on, F.dtype);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> async-proxy reads
        __syncthreads();
      } else if (tid == 0) {
        mbar_wait(&s_bar, 0);  // the bulk store reads what the bulk load wrote (both async proxy)
      }
      if (tid == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(d0), "r"(smem_u32(s_tile)), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // shared memory read before exit
      }
      return;
    }
    // A tile across member boundaries (many small members: Inception V3) whose members
    // are all 16 B aligned: one bulk copy per member piece, issued by the lanes of warp 0
    // (one member each) into the tile's shared memory on one mbarrier; a member's ragged
    // last vector goes element by element.  Misaligned members take the per-vector path.
    __shared__ int s_mis, s_last;
    const int sa = sc.s;
    if (tid < 32) {
      const int sb = seg_of(F, t_end - 1, sa);
      bool mis = false;
      for (int m = sa + (int)tid; m <= sb; m += 32)
        mis |= F.segs[m].count > 0 && ((reinterpret_cast<uintptr_t>(F.src[m]) | reinterpret_cast<uintptr_t>(F.dst[m])) & 15);
      mis = __any_sync(~0u, mis);
      if (tid == 0) {
        s_mis = mis;
        s_last = sb;
      }
    }
    __syncthreads();
    if (!s_mis) {
      const int sb = s_last;
      if (tid < 32) {
        if (tid == 0) {
          mbar_init(&s_bar, 1);
          asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        unsigned bytes = 0;
        for (int m = sa + (int)tid; m <= sb; m += 32) {
          const unsigned long long cnt = F.segs[m].count, v0 = F.segs[m].vbeg, vf = v0 + cnt / VEL;
          const unsigned long long lo = v0 > base ? v0 : base, hi = vf < t_end ? vf : t_end;
          if (hi > lo) {
            tma_load(s_tile + (lo - base), F.src[m] + (lo - v0) * 16, (unsigned)((hi - lo) * 16), &s_bar);
            bytes += (unsigned)((hi - lo) * 16);
          }
          if (cnt % VEL && vf >= base && vf < t_end) {  // ragged last vector
            const unsigned long long left = cnt % VEL;
            Cvt::put(F.dst[m] + (vf - v0) * 16, left,
                     Cvt::slow(F.src[m] + (vf - v0) * 16, left, F.scale, F.scale_on, F.dtype));
          }
        }
        bytes = __reduce_add_sync(~0u, bytes);
        if (tid == 0) mbar_expect_tx(&s_bar, bytes);  // the one arrival: completes with the loads
      }
      if (F.scale_on) {
        __syncthreads();
        mbar_wait(&s_bar, 0);
        for (unsigned long long v = tid; v < t_end - base; v += kSoloThreads)
          s_tile[v] = Pack16<ESZ>::conv(s_tile[v], F.scale, F.scale_on, F.dtype);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
      }
      if (tid < 32) {
        if (!F.scale_on) mbar_wait(&s_bar, 0);
        for (int m = sa + (int)tid; m <= sb; m += 32) {
          const unsigned long long cnt = F.segs[m].count, v0 = F.segs[m].vbeg, vf = v0 + cnt / VEL;
          const unsigned long long lo = v0 > base ? v0 : base, hi = vf < t_end ? vf : t_end;
          if (hi > lo)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         ::"l"(F.dst[m] + (lo - v0) * 16), "r"(smem_u32(s_tile + (lo - base))),
                         "r"((unsigned)((hi - lo) * 16)) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      return;
    }
  }
#endif
  if (fast) {
    constexpr unsigned long long VB = (unsigned long long)VEL * TESZ;  // tensor bytes per wire vector
    const char* gp = g0 + tid * VB;
    char* dp = d0 + tid * VB;
    const unsigned long long nv = t_end - base;
    Raw32 raw[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if ((unsigned long long)u * kSoloThreads + tid < nv) Cvt::load(raw[u], gp + (unsigned long long)u * kSoloThreads * VB);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if ((unsigned long long)u * kSoloThreads + tid < nv)
        Cvt::put(dp + (unsigned long long)u * kSoloThreads * VB, VEL, Cvt::take(raw[u], F.scale, F.scale_on, F.dtype));
    return;
  }
  // member boundary, ragged end or misaligned tensor: per-vector member lookup, the
  // loads of each group of H vectors issued together (memory-level parallelism).
  // The member starts from the tile's first member on are staged in shared memory
  // first: a tile of many small members (Inception V3) would otherwise pay a binary
  // search of dependent global loads for every vector whose member changed.
  __shared__ unsigned long long s_vb[kSoloSegCache];
  const int s0 = sc.s;
  const int nc = F.nseg - s0 < kSoloSegCache ? F.nseg - s0 : kSoloSegCache;
  for (int i = tid; i < nc; i += kSoloThreads) s_vb[i] = F.vbeg[s0 + i];
  __syncthreads();
  // vectors below `vcached` have their member among the staged ones
  const unsigned long long vcached = s0 + nc < F.nseg ? s_vb[nc - 1] : ~0ull;
  constexpr int H = U / 4 > 0 ? U / 4 : 1;
  for (int u0 = 0; u0 < U; u0 += H) {
    Raw32 raw[H];
    uintptr_t gp[H], dp[H];
    unsigned long long left[H];
    bool fast[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const unsigned long long v = base + (unsigned long long)(u0 + h) * kSoloThreads + tid;
      left[h] = 0;
      fast[h] = false;
      if (v < t_end) {
        if (v < vcached) seg_lookup_staged<TESZ>(F, v, sc, s_vb, s0, nc);
        else seg_lookup<TESZ>(F, v, sc);
        const unsigned long long e = v * VEL;
        left[h] = sc.end_el > e ? sc.end_el - e : 0;  // 0: padding after a member
        gp[h] = sc.g + e * TESZ;
        dp[h] = sc.d + e * TESZ;
        fast[h] = left[h] && Cvt::fast(reinterpret_cast<const char*>(gp[h]), left[h]);
        if (fast[h]) Cvt::load(raw[h], reinterpret_cast<const char*>(gp[h]));
      }
    }
#pragma unroll
    for (int h = 0; h < H; ++h) {
      if (left[h] == 0) continue;
      const uint4 x = fast[h] ? Cvt::take(raw[h], F.scale, F.scale_on, F.dtype)
                              : Cvt::slow(reinterpret_cast<const char*>(gp[h]), left[h], F.scale, F.scale_on, F.dtype);
      Cvt::put(reinterpret_cast<char*>(dp[h]), left[h], x);
    }
  }
}

template <class Op, int TESZ>
static cudaError_t launch_solo_t(const FusedParams& p, int nlocal, cudaStream_t s) {
  constexpr int VEL = 16 / Op::kEsz;
  constexpr unsigned long long TILE = (unsigned long long)kSoloThreads * (TESZ > Op::kEsz ? (kSoloU + 1) / 2 : kSoloU);
  unsigned long long tiles = 0;
  for (int b = 0; b < p.nbuf; ++b)
    tiles += p.bufs[b].stile ? p.bufs[b].nstile : ((p.bufs[b].L + VEL - 1) / VEL + TILE - 1) / TILE;
  if (p.solo_tpc > 1) tiles = (tiles + p.solo_tpc - 1) / p.solo_tpc;
  if (tiles == 0) return cudaSuccess;
  if (tiles > 0x7fffffffull) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)tiles, nlocal);
  cfg.blockDim = dim3(kSoloThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ++g_launched;
  return cudaLaunchKernelEx(&cfg, solo_kernel<Op, TESZ>, p);
}

cudaError_t launch_solo(const FusedParams& p, int dtype, int nlocal, cudaStream_t s) {
  const int td = p.tdtype ? p.tdtype : dtype;
  if (td == dtype) {
    switch (dtype) {
      case 1: return launch_solo_t<OpF32, 4>(p, nlocal, s);
      case 2: return launch_solo_t<OpBF16, 2>(p, nlocal, s);
      case 3: return launch_solo_t<OpI32, 4>(p, nlocal, s);
      case 4: return launch_solo_t<OpI64, 8>(p, nlocal, s);
      default: return cudaErrorInvalidValue;
    }
  }
  if (dtype == 2 && td == 1) return launch_solo_t<OpBF16, 4>(p, nlocal, s);
  if (dtype == 1 && td == 2) return launch_solo_t<OpF32, 2>(p, nlocal, s);
  return cudaErrorInvalidValue;
}

template <class Op, int TESZ>
static cudaError_t launch_fused_t(const FusedParams& p, int nch, int nlocal, int threads, cudaStream_t s) {
  const size_t smem = (size_t)p.cache_segs * 8 + fused_smem_bytes(kFusedSmemSegs + 1, threads);
  static bool attr_set[kMaxDevices] = {};  // function attributes are per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= kMaxDevices) return cudaErrorInvalidDevice;
  if (!attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(fused_allreduce_kernel<Op, TESZ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)fused_smem_bytes(kFusedSmemSegs, kMaxRingThreads));
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nch, nlocal);
  cfg.blockDim = dim3(threads + 32 * (p.ring.sig_warps + p.ring.watcher));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  // the CTAs of virtual ranks wait on each other: co-residency is required; a launch of
  // one local rank has no dependency between its own CTAs (each channel talks to the same
  // channel of the neighbouring GPUs), so it may drop the cooperative launch for PDL
  if (p.ring.pdl != 2 || nlocal > 1) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
  }
  if (p.ring.pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  ++g_launched;
  return cudaLaunchKernelEx(&cfg, fused_allreduce_kernel<Op, TESZ>, p);
}

// dtype = wire (fusion buffer / ring) dtype; p.tdtype = tensor dtype (R14)
cudaError_t launch_fused(const FusedParams& p, int dtype, int nch, int nlocal, int threads, cudaStream_t s) {
  const int td = p.tdtype ? p.tdtype : dtype;
  if (td == dtype) {
    switch (dtype) {
      case 1: return launch_fused_t<OpF32, 4>(p, nch, nlocal, threads, s);
      case 2: return launch_fused_t<OpBF16, 2>(p, nch, nlocal, threads, s);
      case 3: return launch_fused_t<OpI32, 4>(p, nch, nlocal, threads, s);
      case 4: return launch_fused_t<OpI64, 8>(p, nch, nlocal, threads, s);
      default: return cudaErrorInvalidValue;
    }
  }
  if (dtype == 2 && td == 1) return launch_fused_t<OpBF16, 4>(p, nch, nlocal, threads, s);
  if (dtype == 1 && td == 2) return launch_fused_t<OpF32, 2>(p, nch, nlocal, threads, s);
  return cudaErrorInvalidValue;
}

template <class Op>
static cudaError_t launch_copy_t(const FusedParams& p, int nch, int nlocal, int threads, cudaStream_t s) {
  const size_t smem = fused_smem_bytes(p.nseg, threads);
  static bool attr_set[kMaxDevices] = {};  // function attributes are per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= kMaxDevices) return cudaErrorInvalidDevice;
  if (!attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(copy_collective_kernel<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)fused_smem_bytes(kFusedSmemSegs, kMaxRingThreads));
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nch, nlocal);
  cfg.blockDim = dim3(threads + 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ++g_launched;
  return cudaLaunchKernelEx(&cfg, copy_collective_kernel<Op>, p);
}

// Copy collectives only move bytes: dispatch on the element size.
cudaError_t launch_copy(const FusedParams& p, int dtype, int nch, int nlocal, int threads, cudaStream_t s) {
  switch (elem_size(dtype)) {
    case 4: return launch_copy_t<OpI32>(p, nch, nlocal, threads, s);
    case 2: return launch_copy_t<OpBF16>(p, nch, nlocal, threads, s);
    case 8: return launch_copy_t<OpI64>(p, nch, nlocal, threads, s);
    default: return cudaErrorInvalidValue;
  }
}

template <class Op>
static cudaError_t launch_pull_t(const FusedParams& p, int nch, int nlocal, int threads, cudaStream_t s) {
  const size_t smem = pull_smem_bytes(p.nseg);
  static bool attr_set[kMaxDevices] = {};  // function attributes are per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= kMaxDevices) return cudaErrorInvalidDevice;
  if (!attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(pull_allreduce_kernel<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)pull_smem_bytes(kFusedSmemSegs));
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nch, nlocal);
  cfg.blockDim = dim3(threads + 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ++g_launched;
  return cudaLaunchKernelEx(&cfg, pull_allreduce_kernel<Op>, p);
}

cudaError_t launch_pull(const FusedParams& p, int dtype, int nch, int nlocal, int threads, cudaStream_t s) {
  switch (dtype) {
    case 1: return launch_pull_t<OpF32>(p, nch, nlocal, threads, s);
    case 2: return launch_pull_t<OpBF16>(p, nch, nlocal, threads, s);
    case 3: return launch_pull_t<OpI32>(p, nch, nlocal, threads, s);
    case 4: return launch_pull_t<OpI64>(p, nch, nlocal, threads, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t pull_max_ctas_per_sm(int dtype, int threads, int* out) {
  const size_t smem = pull_smem_bytes(kFusedSmemSegs);
  switch (dtype) {
    case 1: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, pull_allreduce_kernel<OpF32>, threads + 32, smem);
    case 2: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, pull_allreduce_kernel<OpBF16>, threads + 32, smem);
    case 3: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, pull_allreduce_kernel<OpI32>, threads + 32, smem);
    case 4: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, pull_allreduce_kernel<OpI64>, threads + 32, smem);
    default: return cudaErrorInvalidValue;
  }
}

template <class Op>
static cudaError_t launch_ll_t(const FusedParams& p, int nch, int nlocal, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nch, nlocal);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;  // CTAs of all ranks wait on each other's words
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = p.ring.ll_pdl ? 2 : 1;
  ++g_launched;
  return cudaLaunchKernelEx(&cfg, ll_allreduce_kernel<Op>, p);
}

template <class Op>
static cudaError_t launch_ll128_t(const FusedParams& p, int nch, int nlocal, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nch, nlocal);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;  // CTAs of all ranks wait on each other's lines
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = p.ring.ll_pdl ? 2 : 1;
  ++g_launched;
  return cudaLaunchKernelEx(&cfg, ll128_allreduce_kernel<Op>, p);
}

cudaError_t launch_ll128(const FusedParams& p, int dtype, int nch, int nlocal, cudaStream_t s) {
  switch (dtype) {
    case 1: return launch_ll128_t<OpF32>(p, nch, nlocal, s);
    case 2: return launch_ll128_t<OpBF16>(p, nch, nlocal, s);
    case 3: return launch_ll128_t<OpI32>(p, nch, nlocal, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_ll(const FusedParams& p, int dtype, int nch, int nlocal, cudaStream_t s) {
  switch (dtype) {
    case 1: return launch_ll_t<OpF32>(p, nch, nlocal, s);
    case 2: return launch_ll_t<OpBF16>(p, nch, nlocal, s);
    case 3: return launch_ll_t<OpI32>(p, nch, nlocal, s);
    default: return cudaErrorInvalidValue;
  }
}

// Co-resident LL CTAs per SM, the minimum over the dtype instantiations.
cudaError_t ll_max_ctas_per_sm(int* out) {
  int a = 0, b = 0, c = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, ll_allreduce_kernel<OpF32>, 256, 0);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, ll_allreduce_kernel<OpBF16>, 256, 0);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, ll_allreduce_kernel<OpI32>, 256, 0);
  int d = 0, f = 0, h = 0;  // the LL128 kernels share the budget
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d, ll128_allreduce_kernel<OpF32>, 256, 0);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&f, ll128_allreduce_kernel<OpBF16>, 256, 0);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&h, ll128_allreduce_kernel<OpI32>, 256, 0);
  int m = a < b ? (a < c ? a : c) : (b < c ? b : c);
  m = m < d ? m : d;
  m = m < f ? m : f;
  *out = m < h ? m : h;
  return e;
}

template <class K>
static cudaError_t occupancy_big_smem(int* out, K kernel, int block, size_t smem, size_t max_smem) {
  // the opt-in shared-memory limit is a per-device function attribute: set it on the
  // current device before asking (the answer is 0 blocks without it)
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, kernel, block, smem);
}

cudaError_t fused_max_ctas_per_sm(int dtype, int threads, int* out) {
  const size_t smem = fused_smem_bytes(kFusedSmemSegs, threads);
  const size_t mx = fused_smem_bytes(kFusedSmemSegs, kMaxRingThreads);
  switch (dtype) {
    case 1: return occupancy_big_smem(out, fused_allreduce_kernel<OpF32, 4>, threads + 32, smem, mx);
    case 2: return occupancy_big_smem(out, fused_allreduce_kernel<OpBF16, 2>, threads + 32, smem, mx);
    case 3: return occupancy_big_smem(out, fused_allreduce_kernel<OpI32, 4>, threads + 32, smem, mx);
    case 4: return occupancy_big_smem(out, fused_allreduce_kernel<OpI64, 8>, threads + 32, smem, mx);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t ring_max_ctas_per_sm(int dtype, int threads, int* out) {
  switch (dtype) {
    case 1: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, ring_allreduce_kernel<OpF32>, threads + 32, 0);
    case 2: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, ring_allreduce_kernel<OpBF16>, threads + 32, 0);
    case 3: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, ring_allreduce_kernel<OpI32>, threads + 32, 0);
    case 4: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, ring_allreduce_kernel<OpI64>, threads + 32, 0);
    default: return cudaErrorInvalidValue;
  }
}


// ------------------------------------------------------------------ bulk-copy push ring launchers
size_t bulk_smem_bytes(int stages, int stage_bytes, bool two) {
  return (size_t)stages * ((two ? 2 : 1) * (size_t)stage_bytes + sizeof(StageDesc) + 3 * sizeof(unsigned long long));
}

template <class Op>
static cudaError_t launch_bulk_t(const FusedParams& p, int nch, int nlocal, cudaStream_t s) {
  const bool ring = p.ring.N > 1;
  const size_t smem = bulk_smem_bytes(p.bulk_stages, p.bulk_stage_bytes, ring);
  cudaError_t e = cudaFuncSetAttribute(bulk_allreduce_kernel<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nch, nlocal);
  cfg.blockDim = dim3(kBulkThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  if (ring) {
    attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (they wait on each other)
    attr[0].val.cooperative = 1;
  } else {
    // N = 1: CTAs wait on nothing but the previous grid (griddepcontrol.wait)
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ++g_launched;
  return cudaLaunchKernelEx(&cfg, bulk_allreduce_kernel<Op>, p);
}

cudaError_t launch_bulk(const FusedParams& p, int dtype, int nch, int nlocal, cudaStream_t s) {
  switch (dtype) {
    case 1: return launch_bulk_t<OpF32>(p, nch, nlocal, s);
    case 2: return launch_bulk_t<OpBF16>(p, nch, nlocal, s);
    case 3: return launch_bulk_t<OpI32>(p, nch, nlocal, s);
    case 4: return launch_bulk_t<OpI64>(p, nch, nlocal, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t bulk_max_ctas_per_sm(int dtype, int stages, int stage_bytes, int* out, bool two) {
  const size_t smem = bulk_smem_bytes(stages, stage_bytes, two);
  cudaError_t e = cudaSuccess;
  switch (dtype) {
    case 1:
      e = cudaFuncSetAttribute(bulk_allreduce_kernel<OpF32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, bulk_allreduce_kernel<OpF32>, kBulkThreads, smem);
      return e;
    case 2:
      e = cudaFuncSetAttribute(bulk_allreduce_kernel<OpBF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, bulk_allreduce_kernel<OpBF16>, kBulkThreads, smem);
      return e;
    case 3:
      e = cudaFuncSetAttribute(bulk_allreduce_kernel<OpI32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, bulk_allreduce_kernel<OpI32>, kBulkThreads, smem);
      return e;
    case 4:
      e = cudaFuncSetAttribute(bulk_allreduce_kernel<OpI64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, bulk_allreduce_kernel<OpI64>, kBulkThreads, smem);
      return e;
    default: return cudaErrorInvalidValue;
  }
}


cudaError_t launch_ll128_selftest(const RingParams& p, int nch, int nlocal, int rounds, int lines_per_cta,
                                  unsigned long long* torn, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nch, nlocal);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // virtual ranks: readers and writers co-resident
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, ll128_selftest_kernel, p, rounds, lines_per_cta, torn);
}

}  // namespace hvd

// Internal types shared by the host runtime (hvd_runtime.cpp) and the
// sm_100a kernels (hvd_kernels.cu).  Not part of the ABI (include/hvd.h is).
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace hvd {

constexpr int kMaxLocal = 8;        // virtual ranks per comm (one launch spans them all)
constexpr int kMaxChannels = 256;   // ring CTAs per rank
constexpr int kMemberAlign = 16;    // fusion-buffer member alignment, bytes (R2)
constexpr int kChunkQuantum = 256;  // chunk-boundary quantum, bytes (R2)
constexpr int kPackVecBytes = 16;   // pack/unpack vector (== kMemberAlign, so a vector never
                                    // spans two members)

inline int elem_size(int dtype) {
  switch (dtype) {
    case 1: return 4;  // HVD_FLOAT32
    case 2: return 2;  // HVD_BFLOAT16
    case 3: return 4;  // HVD_INT32
    case 4: return 8;  // HVD_INT64
    default: return 0;
  }
}

// ---------------------------------------------------------------- job timeline
// Horovod Timeline ("what each node was doing at each time step throughout
// a training job"): every kernel launch of a comm with the job timeline on records, per
// local rank, its first CTA's start and its last CTA's end (%globaltimer, ns).  CTAs
// fold into a device record of the launch; the last CTA of a local rank copies the
// result into a host-mapped slot (kJtWords words, seq written last) and re-arms the
// device record, so the host drains finished launches without synchronising.
constexpr int kJtSlots = 4096;   // launches in flight before a slot is reused
constexpr int kJtWords = 4;      // device: {begin (min), end (max), CTAs done, 0}; host: {seq, begin, end, ctas}
struct JtRef {
  unsigned long long* rec;       // device record of this launch: [kMaxLocal][kJtWords] (nullptr = off)
  unsigned long long* host;      // host-mapped slot of this launch: [kMaxLocal][kJtWords]
  unsigned long long seq;        // launch sequence number (1-based)
};

// ---------------------------------------------------------------- ring kernel
// One ring rank as seen by the kernel: its own buffers and its successor's.
struct RingRank {
  char* buf;                     // fusion buffer (capacity bytes)
  char* scratch;                 // reduce-scatter receive scratch (capacity bytes)
  char* scratch1;                // second receive half: a channel alternates halves per buffer
  unsigned long long* flags;     // [kMaxChannels] written by the predecessor
  unsigned long long* stats;     // [2] sent bytes, sent chunk messages
  char* nbuf;                    // successor's fusion buffer (peer / same-device)
  char* nscratch;                // successor's scratch
  char* nscratch1;               // successor's second half
  unsigned long long* nflags;    // successor's flags
  unsigned long long* rflags;    // [kMaxChannels] ready flags, written by the successor (handshake)
  unsigned long long* pready;    // predecessor's ready flags (this rank writes them)
  unsigned long long* rhash;     // [kMaxChannels] call hashes, written by the successor
  unsigned long long* phash;     // predecessor's call hashes (this rank writes them)
  // pull protocol (pull_allreduce_kernel)
  char* pull[2];                 // own pull buffers (call parity), read by the successor
  const char* ppull[2];          // predecessor's pull buffers
  unsigned long long* pflags_own;   // [kMaxChannels] own progress (read remotely by the successor)
  const unsigned long long* pflags_pred;  // predecessor's progress
  unsigned long long* done_own;  // calls completed by this rank (read remotely by the predecessor)
  const unsigned long long* done_succ;  // successor's completed calls
  unsigned long long* exits;     // CTA exit counter of this rank (local)
  unsigned long long* ll;        // LL region (small-buffer protocol), written by the predecessor
  unsigned long long* nll;       // successor's LL region
  int rank;                      // ring rank
  int pad;
};

enum RingMode : int {
  kRingAllreduce = 0,   // N-1 reduce-scatter + N-1 all-gather iterations
  kRingAllgather = 1,   // N-1 all-gather iterations, blocks of `q` elements per rank
  kRingBroadcast = 2,   // pipelined forward root -> root+1 -> ...
};

struct RingParams {
  RingRank rk[kMaxLocal];
  unsigned long long base[kMaxChannels];  // signal counter value before this call
  unsigned long long L;         // elements in the buffer
  unsigned long long q;         // chunk length, elements (multiple of the quantum)
  unsigned long long ch_el;     // elements per channel per chunk (multiple of the quantum)
  unsigned long long slice_el;  // elements per pipelining slice (multiple of the quantum)
  int N;                        // ring size
  int K;                        // slices per channel per chunk
  int mode;                     // RingMode
  int root;                     // broadcast root
  int* err;                     // host-mapped error word (device address)
  unsigned long long timeout_ns;
  int sig_mode;                 // signal fence variant (hvd_kernels.cu signal_loop)
  int sig_warps;                // fused: signal warps per CTA (1: signal_loop, > 1: signal_loop_multi)
  int tl_max;                   // timeline: slice records per channel (0 = timeline off)
  unsigned long long* tl;       // timeline records of this launch (per local rank, see tl_words)
  int window;                   // fused: max pushed-but-unfenced slices per channel (0 = no limit)
  int fin_lag;                  // fused: final-scatter interleave lag in slices
  unsigned long long epoch;     // ring/fused/copy: handshake epoch of this launch (LL: flag)
  unsigned long long hash;      // ring/fused: hash of the call's geometry (HVD_ERR_MISMATCH)
  int parity;                   // pull protocol: pull buffer of this call
  int call;                     // pull protocol: 1-based call index
  unsigned long long exits_target;  // pull protocol: cumulative CTA exits after this call
  int watcher;                  // fused: dependency watcher lane (HVD_CFG_WATCHER)
  int preissue;                 // fused: gather loads before the dependency wait (HVD_CFG_PREISSUE)
  int ll_pdl;                   // LL / LL128: programmatic dependent launch (HVD_CFG_LL_PDL)
  int pdl;                      // fused: programmatic dependent launch (HVD_CFG_FUSED_PDL: 0 off,
                                //   1 with the cooperative launch, 2 instead of it; one local rank only)
  unsigned pace_cyc;            // fused: ns per row of remote stores per channel (0 = unpaced)
  unsigned pace_burst;          // fused: credit a paced channel may build up while idle, ns
  JtRef jt;                     // job timeline record of this launch
};

// Timeline buffer of one local rank (Horovod Timeline): for every
// channel, tl_max data records {t_begin, t_end} (ns, %globaltimer) of its slice
// operations in program order, then tl_max signal records {t_publish, count}.
__host__ __device__ inline size_t tl_words(int tl_max) { return (size_t)kMaxChannels * tl_max * 4; }

// Signals each channel sends per call (host keeps the per-channel base in step).
inline unsigned long long ring_signals(int mode, int N, int K) {
  if (N <= 1) return 0;
  if (mode == kRingAllreduce) return 2ull * (N - 1) * K;
  if (mode == kRingBroadcast) return (unsigned long long)K;
  return 1ull * (N - 1) * K;
}

// ---------------------------------------------------------------- pack / unpack
struct PackSeg {
  unsigned long long dst_off;   // element offset in the fusion buffer (16 B aligned)
  unsigned long long count;     // elements
  unsigned long long vbeg;      // first 16 B vector of the member in the buffer
  unsigned long long pad;
};

struct PackParams {
  const PackSeg* segs;          // [nseg]
  char* const* src;             // [nlocal * nseg] tensor addresses (already + src_off)
  const int* tile_seg;          // [ntiles + 1] segment of each tile's first vector (+ last)
  char* buf[kMaxLocal];         // fusion buffer per local rank
  unsigned long long nvec;      // 16 B vectors in the buffer
  unsigned long long tile_vecs; // vectors per tile
  unsigned long long ntiles;
  int nseg;
  int scale_on;                 // 1: multiply by `scale` (AVERAGE)
  float scale;                  // fl32(1/N)
  int pad;
  JtRef jt;                     // job timeline record of this launch
};

// N = 1 (solo_kernel): tiles of at most kSoloTileVecs 16 B vectors that never cross a
// member, built with the plan (same-dtype buffers, one local rank).  A tile either moves
// `bytes` (whole vectors) from src to dst by bulk copies plus `ragged` elements of the
// member's partial last vector after them, or (flags & 1: a misaligned member) covers the
// buffer vectors [src, dst) through the per-vector member lookup.
#ifndef HVD_SOLO_THREADS
#define HVD_SOLO_THREADS 128
#endif
#ifndef HVD_SOLO_U
#define HVD_SOLO_U 4  // 8 KiB tiles (profiles/r02_solo_tile_sweep/: vs 16 KiB, 64 MiB 0.938 -> 0.945 of HBM,
                      // Inception V3 fp32 0.835 -> 0.848, bf16 0.666 -> 0.712; 4 KiB tiles lose on the model sets)
#endif
constexpr unsigned long long kSoloTileVecs = (unsigned long long)HVD_SOLO_THREADS * HVD_SOLO_U;
#ifndef HVD_SOLO_TPC
#define HVD_SOLO_TPC 1  // member tiles per CTA when every tile of a launch is a plain bulk copy
#endif
constexpr int kSoloTPC = HVD_SOLO_TPC;
struct SoloTile {
  unsigned long long src, dst;
  unsigned bytes, ragged, flags, member;
};

// One fusion buffer of a multi-buffer fused launch (geometry + member tables).
struct BufDesc {
  const PackSeg* segs;               // [nseg]
  char* const* src;                  // [nlocal * nseg] gather addresses
  char* const* dst;                  // [nlocal * nseg] scatter addresses
  char* const* rdst;                 // [nlocal * nseg] registered: successor's addresses
  const unsigned long long* vbeg;    // [nseg] member start vectors
  const int* tile_seg;               // [L / tile_vecs + 2] member of vector p * tile_vecs (+ last member):
  unsigned long long tile_vecs;      //   bounds the member search of any vector to [tile_seg[p], tile_seg[p+1]]
  unsigned long long L, q, ch_el, slice_el;
  int nseg, K;
  int owner;                         // fused: -1 = every channel takes a share; else the first
                                     //  of the nch consecutive channels (mod grid) that run it
  int nch;                           // fused: channels of this buffer; LL: its CTAs
  unsigned ll_off;                   // LL: word offset of this buffer's slots in a parity half
  int pad;
  const SoloTile* stile;             // N = 1: member tiles (nullptr: tiles over the buffer's vectors)
  unsigned long long nstile;
};
constexpr int kMaxMultiBufs = 96;    // fusion buffers per fused launch (kernel parameter space)

// Fused zero-copy allreduce of one fusion buffer (pack + ring + unpack in one launch).
constexpr int kFusedSmemSegs = 4096;  // member-offset table cached in shared memory up to this size
#ifndef HVD_PIPE
#define HVD_PIPE 8
#endif
constexpr int kPipe = HVD_PIPE;       // cp.async prefetch depth (rows of 16 B per data thread)
constexpr int kMaxRingThreads = 384;  // data threads per ring / fused CTA
inline size_t pull_smem_bytes(int nseg) {
  const size_t vb = nseg <= kFusedSmemSegs ? (size_t)(nseg + 15) / 16 * 16 * 8 : 0;
  return vb + 6ull * (16 << 10);  // + kStages x kStageBytes (hvd_kernels.cu)
}
inline size_t fused_smem_bytes(int nseg, int threads) {
  const size_t vb = nseg <= kFusedSmemSegs ? (size_t)(nseg + 1) / 2 * 2 * 8 : 0;
  return vb + 3ull * kPipe * threads * 16;  // slots0: 32 B per row (wire conversion), slots1: 16 B
}
struct FusedParams {
  RingParams ring;
  const PackSeg* segs;               // [nseg]
  char* const* src;                  // [nlocal * nseg] gather addresses
  char* const* dst;                  // [nlocal * nseg] scatter addresses (nullptr: same as src)
  const unsigned long long* vbeg_global;  // [nseg] (used when nseg > kFusedSmemSegs)
  int nseg;
  int scale_on;
  float scale;
  int dtype;                         // wire dtype (fusion buffer / ring)
  int tdtype;                        // tensor dtype (0: same as dtype)
  int registered;                    // 1: all-gather writes into the successor's tensors (rdst)
  char* const* rdst;                 // [nlocal * nseg] successor's tensor addresses (registered)
  // multi-buffer fused kernel
  int nbuf;
  int cache_segs;                    // member-offset cache entries in shared memory
  unsigned long long region_el;      // channel-private region of scratch / buffer, elements
  // bulk-copy push kernel (bulk_allreduce_kernel)
  int bulk_stages;                   // shared-memory stages per CTA
  int bulk_stage_bytes;              // bytes per stage (multiple of 16)
  int bulk_depth;                    // bulk store groups left incomplete before retiring a stage
  int solo_tpc;                      // N = 1 member tiles per CTA (solo_kernel; 1 = one)
  BufDesc bufs[kMaxMultiBufs];
};

// Launchers (hvd_kernels.cu).  All return a cudaError_t.
cudaError_t launch_fused(const FusedParams& p, int dtype, int nch, int nlocal, int threads, cudaStream_t s);
cudaError_t launch_copy(const FusedParams& p, int dtype, int nch, int nlocal, int threads, cudaStream_t s);
cudaError_t launch_pull(const FusedParams& p, int dtype, int nch, int nlocal, int threads, cudaStream_t s);
cudaError_t launch_ll(const FusedParams& p, int dtype, int nch, int nlocal, cudaStream_t s);
constexpr unsigned long long kLLMaxBytes = 256ull << 10;  // default LL payload limit for a lone buffer
constexpr unsigned long long kLLLimitBytes = 8ull << 20;  // largest HVD_CFG_LL_MAX_BYTES accepted
constexpr unsigned long long kLL128LimitBytes = 64ull << 20;  // largest HVD_CFG_LL128_MAX_BYTES accepted
// LL region of a rank: [LL half 0][LL half 1][LL128 half 0][LL128 half 1].  LL and
// LL128 never share memory: an LL word is taken when its upper 32 bits equal the epoch,
// and LL128 lines carry raw data there (stale LL128 data must never be
// polled by LL).  Launches of either protocol alternate the halves of their own pair.
// LL: (2N-2) steps x chunk slot of 2 q esz bytes (8 B word per 4 B of data) per half
// = 4 (N-1) q esz < 4 L + 4 (N-1) N 256 <= 32.1 MiB for L <= kLLLimitBytes.
// LL128: 2 (N-1) x lines x 128 B per half ~ 2 (N-1)/N x 8/7 x L <= 2.3 L: 160 MiB
// halves hold a 64 MiB buffer at any N <= 8.
constexpr unsigned long long kLLHalfBytes = 48ull << 20;
constexpr unsigned long long kLL128HalfBytes = 160ull << 20;
constexpr unsigned long long kLLRegionBytes = 2 * (kLLHalfBytes + kLL128HalfBytes);
cudaError_t pull_max_ctas_per_sm(int dtype, int threads, int* out);
cudaError_t ll_max_ctas_per_sm(int* out);
cudaError_t launch_ll128(const FusedParams& p, int dtype, int nch, int nlocal, cudaStream_t s);
cudaError_t launch_ll128_selftest(const RingParams& p, int nch, int nlocal, int rounds, int lines_per_cta,
                                  unsigned long long* torn, cudaStream_t s);
cudaError_t launch_bulk(const FusedParams& p, int dtype, int nch, int nlocal, cudaStream_t s);
cudaError_t bulk_max_ctas_per_sm(int dtype, int stages, int stage_bytes, int* out, bool two = true);
size_t bulk_smem_bytes(int stages, int stage_bytes, bool two = true);  // two: A and B stages (N > 1)
cudaError_t launch_solo(const FusedParams& p, int dtype, int nlocal, cudaStream_t s);
cudaError_t fused_max_ctas_per_sm(int dtype, int threads, int* out);
cudaError_t launch_pack(const PackParams& p, int dtype, int nlocal, int grid, int threads,
                        cudaStream_t s);
cudaError_t launch_unpack(const PackParams& p, int dtype, int nlocal, int grid, int threads,
                          cudaStream_t s);
cudaError_t launch_scale(char* const* bufs, int nlocal, unsigned long long count, int dtype,
                         float scale, int grid, int threads, const JtRef& jt, cudaStream_t s);
unsigned long long kernels_launched();  // launches issued by the launchers above (monotone)
cudaError_t launch_jt_clock(unsigned long long* host_out, cudaStream_t s);  // %globaltimer -> host word
cudaError_t launch_ring(const RingParams& p, int dtype, int nch, int nlocal, int threads,
                        cudaStream_t s);
cudaError_t ring_max_ctas_per_sm(int dtype, int threads, int* out);

}  // namespace hvd

// Host runtime behind the C ABI (include/hvd.h): communicator, buffers, CUDA-IPC
// peer mapping, plan cache with device-resident segment tables, and the
// stream-ordered enqueue of pack -> ring -> unpack per fusion buffer
// (§7 steps 2-6).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <string>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <list>
#include <vector>

#include <dlfcn.h>
#include <unistd.h>

#include "../../include/hvd.h"
#include "hvd_internal.h"
#include "hvd_plan.h"
#include "hvd_negotiate.h"
#include "hvd_jobtrace.h"

using namespace hvd;

namespace {

constexpr uint64_t kDefaultFusionBytes = 64ull << 20;  // P:L368-369 "Default ... 64 MB" (R9)
constexpr uint64_t kTailBytes = 16384;  // flags, stats, ready flags, pull progress, done/exit counters
constexpr uint32_t kBlobMagic = 0x48564442u;            // "HVDB"
constexpr int kPackThreads = 256;
constexpr size_t kBulkMaxSmem = 227 << 10;  // dynamic shared memory of one bulk-push CTA
constexpr int kPackVecsPerThread = 8;
constexpr size_t kPlanCacheSize = 32;

struct Blob {
  uint32_t magic;
  int32_t version;
  int32_t rank, size, device, pid;
  uint64_t capacity;
  uint64_t region_bytes;
  cudaIpcMemHandle_t handle;
  char pci[32];  // PCI bus id of the rank's GPU (NVLink check of the ring links)
  uint64_t region_addr;  // region address in the owner process (a rank in the SAME process
                         // maps it by peer access: CUDA IPC cannot open its own handles)
  int32_t has_pull, pad;       // pull protocol buffers allocated (HVD_CFG_PULL_BUFFERS)
  cudaIpcMemHandle_t pull_handle;
  uint64_t pull_addr;
};

struct DevPlanBuffer {
  int dtype;                            // buffer (wire) dtype
  int tdtype = 0;                       // tensor dtype
  uint64_t L;
  PackParams pp;                        // device pointers filled in
  const unsigned long long* vbeg;       // [nseg] member start vectors (fused kernel, large plans)
  char* const* dst = nullptr;           // [nlocal * nseg] scatter addresses (nullptr: = pp.src)
  char* const* rdst = nullptr;          // [nlocal * nseg] registered: successor's addresses
  const SoloTile* stile = nullptr;      // N = 1: member tiles (solo_kernel)
  uint64_t nstile = 0;
  bool stile_slow = false;              // some member tile takes the per-vector path
};

// A registered tensor list (hvd_register): this rank's tensors plus the successor's
// same-index tensors mapped into this process (CUDA IPC), so the all-gather steps
// can write final values straight into the successor's tensors.
struct Registration {
  int n = 0;
  std::vector<hvd_tensor> own;     // [nlocal * n]
  std::vector<char*> succ;         // [nlocal * n] successor's tensor addresses
  bool live = false;
};

struct CachedPlan {
  std::vector<uint64_t> key;
  std::vector<DevPlanBuffer> bufs;
  void* dmem = nullptr;
  void* hmem = nullptr;
};

}  // namespace

struct hvd_comm {
  int rank = 0, size = 1, device = 0, nlocal = 1;
  bool virt = false, connected = false, closed = false;
  uint64_t cap = 0;    // fusion capacity (plans, limits)
  uint64_t bufsz = 0;  // bytes of each region buffer (cap + slack)
  char* region[kMaxLocal] = {};
  char* pull_mem[kMaxLocal] = {};  // pull protocol: [pull 0][pull 1], bufsz each (lazy)
  const char* pred_pull = nullptr; // predecessor's pull buffers, real mode
  bool pred_pull_ipc = false;
  bool want_pull = false;          // real mode: allocate pull buffers at hvd_get_ipc_blob
  bool pull_ok = false;            // every rank's pull buffers are mapped: protocol 0 usable
  bool blob_out = false;           // real mode: the IPC blob was exported
  char* peer_region = nullptr;   // successor's region (IPC mapped), real mode
  char* pred_region = nullptr;   // predecessor's region (IPC mapped), real mode
  bool peer_ipc = false, pred_ipc = false;  // mapped by IPC (else: same process, peer access)
  int succ_device = -1;                     // successor's device (same-process registration)
  RingRank rk[kMaxLocal] = {};
  unsigned long long base[kMaxChannels] = {};
  int* err_host = nullptr;
  int* err_dev = nullptr;   // device-memory error words the kernels poll (ErrWords)
  int sm_count = 148;
  // tuning (hvd_set_config)
  int channels = 128;
  int64_t slice_bytes = 0;  // 0 = auto: about half of a channel's share of a chunk, 32..128 KiB
  int threads = 256;  // HVD_CFG_THREADS (256 vs 384: 0.5-1 % faster at N = 2, 4; 98 vs 147 KB smem)
  int64_t timeout_ms = 30000;
  int pack_ctas_per_sm = 8;
  int profile = 0;
  int sig_mode = 1;
  int sig_warps = 1;  // HVD_CFG_SIGNAL_WARPS (fused kernel)
  int fused = 1;
  int multi_bufs = kMaxMultiBufs;  // fusion buffers per fused launch
  int window = 2;  // HVD_CFG_WINDOW (measured: N = 4 +5-8 %, N = 2 neutral)
  int fin_lag = 1;
  unsigned long long hs_epoch = 0;  // copy-collective handshake epochs issued
  unsigned long long ll_epoch = 0;  // LL launches issued (flag value = epoch)
  int64_t ll_max = (int64_t)kLLMaxBytes;  // HVD_CFG_LL_MAX_BYTES
  int ll_ctas = 1;                         // co-resident LL CTAs per local rank
  int64_t ll128_max = 0;                   // HVD_CFG_LL128_MAX_BYTES
  int ll128_status = 0;                    // HVD_CFG_LL128_STATUS (hvd_ll128_selftest)
  int protocol = 1;                 // 0: pull (receiver-initiated TMA loads), 1: push (SM stores),
                                    // 2: bulk push (TMA bulk loads / stores through shared memory)
  int bulk_stages = 6;              // HVD_CFG_BULK_STAGES
  int bulk_stage_bytes = 16 << 10;  // HVD_CFG_BULK_STAGE_BYTES
  int bulk_depth = 1;               // HVD_CFG_BULK_DEPTH
  int bulk_channels = 148;          // HVD_CFG_BULK_CHANNELS
  int64_t bulk_slice = 64 << 10;    // HVD_CFG_BULK_SLICE_BYTES
  int solo_kernel = 0;              // HVD_CFG_SOLO_KERNEL: 1 persistent bulk kernel, 0 tile-per-CTA kernel
  int solo_stages = 6;              // HVD_CFG_SOLO_STAGES
  int solo_stage_bytes = 32 << 10;  // HVD_CFG_SOLO_STAGE_BYTES
  int64_t solo_tail = 0;            // HVD_CFG_SOLO_TAIL: member tiles at a buffer's end cut in half
  int pace_gbps = 0;                // HVD_CFG_PACE_GBPS: fused push remote-store pacing (0 = off)
  int fused_pdl = 0;                // HVD_CFG_FUSED_PDL
  int watcher = 0;                  // HVD_CFG_WATCHER
  int host_zero_copy = 0;           // HVD_CFG_HOST_ZERO_COPY (measured slower: off)
  int preissue = -1;                // HVD_CFG_PREISSUE (-1: on for N > 2, measured +2 % at N = 4)
  int ll_pdl = 1;                   // HVD_CFG_LL_PDL (N = 4 <= 1 MiB: 1-7 % lower latency; N = 2 neutral)
  int pace_burst_rows = 2;          // HVD_CFG_PACE_BURST_ROWS
  int clock_khz = 1965000;          // SM clock (cudaDevAttrClockRate): pacing cycles
  unsigned long long pbase[kMaxChannels] = {};  // pull-protocol progress counter bases
  int pull_calls = 0;
  unsigned long long pull_exits = 0;  // cumulative CTA exits of the pull kernel (per rank)
  std::vector<std::pair<int, int>> occ_cache;  // (kernel/dtype/threads key, CTAs per SM)
  std::vector<Registration> regs;               // hvd_register
  Registration bufreg;                          // hvd_allreduce_buffer: the fusion buffer itself
  std::map<std::string, char*> ipc_maps;        // opened peer allocations (by handle bytes)
  // timeline (HVD_CFG_TIMELINE): device records of the most recent fused launch
  int tl_max = 0;
  unsigned long long* tl = nullptr;
  int tl_nch = 0, tl_K = 0, tl_T = 0, tl_slices = 0, tl_kind = 0;
  JobTrace* jt = nullptr;  // job-wide timeline (HVD_TIMELINE / hvd_timeline_start)
  std::list<CachedPlan> cache;
  // launch statistics (hvd_kernel_stats)
  uint64_t launches[HVD_KERNEL_KINDS] = {};
  struct Timed { int kind; cudaEvent_t a, b; };
  std::vector<Timed> timed;
  std::vector<cudaEvent_t> event_pool;
  // host-buffer allreduce (hvd_allreduce_host): device staging slots + copy streams
  static constexpr int kHostSlots = 3;
  char* stage[kMaxLocal] = {};
  uint64_t stage_chunk = 0;  // bytes per slot
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_in[kHostSlots] = {}, ev_red[kHostSlots] = {}, ev_out[kHostSlots] = {};
  cudaEvent_t ev_start = nullptr, ev_done = nullptr;
};

namespace {
uint64_t solo_tail_tiles(const hvd_comm* c) {
  return c->solo_tail >= 0 ? (uint64_t)c->solo_tail : (uint64_t)c->sm_count * 9;
}
}  // namespace


namespace {

int cuda_fail(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return HVD_OK;
  std::fprintf(stderr, "[hvd] %s: %s\n", what, cudaGetErrorString(e));
  return HVD_ERR_CUDA;
}
#define CK(call)                                    \
  do {                                              \
    int _st = cuda_fail((call), #call);             \
    if (_st != HVD_OK) return _st;                  \
  } while (0)

// Region: [fusion buffer][RS scratch 0][RS scratch 1][tail][LL]; each buffer is
// `bufsz` = kRegionFactor x capacity + slack bytes (the slack absorbs the quantum
// rounding of the channel-private layout).  `cap` arguments below are bufsz.  scratch1
// is the second reduce-scatter receive half (a channel alternates halves buffer by
// buffer).  The pull protocol's two buffers are a separate allocation made only when
// that protocol is enabled (HVD_CFG_PULL_BUFFERS).
constexpr uint64_t kRegionSlack = 2ull << 20;
constexpr uint64_t kRegionFactor = 3;
constexpr uint64_t kNumBufs = 3;
char* buf_of(char* region) { return region; }
char* scratch_of(char* region, uint64_t cap) { return region + cap; }
char* scratch1_of(char* region, uint64_t cap) { return region + 2 * cap; }
unsigned long long* flags_of(char* region, uint64_t cap) {
  return reinterpret_cast<unsigned long long*>(region + kNumBufs * cap);
}
unsigned long long* stats_of(char* region, uint64_t cap) {
  return reinterpret_cast<unsigned long long*>(region + kNumBufs * cap + kMaxChannels * 8);
}
unsigned long long* tail_of(char* region, uint64_t cap) {
  return reinterpret_cast<unsigned long long*>(region + kNumBufs * cap);
}
unsigned long long* rflags_of(char* region, uint64_t cap) { return tail_of(region, cap) + 512; }
unsigned long long* rhash_of(char* region, uint64_t cap) { return tail_of(region, cap) + 768; }
unsigned long long* pflags_of(char* region, uint64_t cap) { return tail_of(region, cap) + 1024; }
unsigned long long* done_of(char* region, uint64_t cap) { return tail_of(region, cap) + 1536; }
unsigned long long* exits_of(char* region, uint64_t cap) { return tail_of(region, cap) + 1537; }
unsigned long long* ll_of(char* region, uint64_t cap) {
  return reinterpret_cast<unsigned long long*>(region + kNumBufs * cap + kTailBytes);
}

int common_init(hvd_comm* c, uint64_t fusion_bytes) {
  c->cap = ((fusion_bytes ? fusion_bytes : kDefaultFusionBytes) + 4095) / 4096 * 4096;
  // region buffers hold kRegionFactor fusion buffers: the buffers of a multi-buffer call
  // then fit side by side in the channel-private layout and run concurrently
  c->bufsz = (c->cap <= (256ull << 20) ? kRegionFactor : 1) * c->cap + kRegionSlack;
  CK(cudaSetDevice(c->device));
  CK(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, c->device));
  CK(cudaDeviceGetAttribute(&c->clock_khz, cudaDevAttrClockRate, c->device));
  // error words: the host-mapped one hvd_poll_error reads, and the device-memory one the
  // kernels poll (hvd_kernels.cu ErrWords: {code, pad, host-mapped address})
  CK(cudaHostAlloc(reinterpret_cast<void**>(&c->err_host), sizeof(int), cudaHostAllocMapped));
  *c->err_host = 0;
  int* err_mapped = nullptr;
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&err_mapped), c->err_host, 0));
  {
    struct { int code, pad; int* host; } words = {0, 0, err_mapped};
    CK(cudaMalloc(reinterpret_cast<void**>(&c->err_dev), sizeof(words)));
    CK(cudaMemcpy(c->err_dev, &words, sizeof(words), cudaMemcpyHostToDevice));
  }
  const uint64_t region_bytes = kNumBufs * c->bufsz + kTailBytes + kLLRegionBytes;
  for (int l = 0; l < c->nlocal; ++l) {
    CK(cudaMalloc(reinterpret_cast<void**>(&c->region[l]), region_bytes));
    CK(cudaMemset(c->region[l] + kNumBufs * c->bufsz, 0, kTailBytes + kLLRegionBytes));
    RingRank& r = c->rk[l];
    const uint64_t bz = c->bufsz;
    r.buf = buf_of(c->region[l]);
    r.scratch = scratch_of(c->region[l], bz);
    r.scratch1 = scratch1_of(c->region[l], bz);
    r.flags = flags_of(c->region[l], bz);
    r.stats = stats_of(c->region[l], bz);
    r.rflags = rflags_of(c->region[l], bz);
    r.rhash = rhash_of(c->region[l], bz);
    r.pflags_own = pflags_of(c->region[l], bz);
    r.done_own = done_of(c->region[l], bz);
    r.exits = exits_of(c->region[l], bz);
    r.ll = ll_of(c->region[l], bz);
    r.rank = c->virt ? l : c->rank;
  }
  int ll_per_sm = 0;
  CK(ll_max_ctas_per_sm(&ll_per_sm));
  c->ll_ctas = std::max(1, std::min(ll_per_sm, 4) * c->sm_count / c->nlocal);
  // Protocol limits for a lone buffer (profiles/r02_ll128_crossover_n{2,4}.json, the 16/15
  // line layout): LL up to 256 KiB, LL128 up to 24 MiB (N = 2) / 48 MiB (N > 2), the fused
  // push beyond (N = 2: LL128 55 vs 58 us at 24 MiB, 71 vs 65 at 32; N = 4: 94 vs 110 us at
  // 32 MiB, a tie at 48, 181 vs 166 at 64; Inception V3 bf16's one 45 MiB buffer thus runs
  // LL128 at N > 2)
  c->ll_max = (int64_t)kLLMaxBytes;
  c->ll128_max = c->size <= 2 ? (int64_t)(24ull << 20) : (int64_t)(48ull << 20);
  CK(cudaDeviceSynchronize());
  return HVD_OK;
}

void set_neighbours(RingRank& r, char* succ_region, char* pred_region, uint64_t cap) {
  r.nbuf = buf_of(succ_region);
  r.nscratch = scratch_of(succ_region, cap);
  r.nscratch1 = scratch1_of(succ_region, cap);
  r.nflags = flags_of(succ_region, cap);
  r.pready = rflags_of(pred_region, cap);
  r.phash = rhash_of(pred_region, cap);
  r.pflags_pred = pflags_of(pred_region, cap);
  r.done_succ = done_of(succ_region, cap);
  r.nll = ll_of(succ_region, cap);
}

// The pull protocol's two buffers (HVD_CFG_PULL_BUFFERS): a separate allocation, made
// only when that protocol is enabled, so the default footprint is the push path's.
int alloc_pull(hvd_comm* c) {
  if (c->pull_mem[0]) return HVD_OK;
  CK(cudaSetDevice(c->device));
  CK(cudaDeviceSynchronize());
  for (int l = 0; l < c->nlocal; ++l) {
    CK(cudaMalloc(reinterpret_cast<void**>(&c->pull_mem[l]), 2 * c->bufsz));
    c->rk[l].pull[0] = c->pull_mem[l];
    c->rk[l].pull[1] = c->pull_mem[l] + c->bufsz;
  }
  if (c->virt) {
    for (int l = 0; l < c->nlocal; ++l)
      for (int p = 0; p < 2; ++p) c->rk[l].ppull[p] = c->rk[(l + c->nlocal - 1) % c->nlocal].pull[p];
    c->pull_ok = true;
  }
  return HVD_OK;
}

bool env_on(const char* name) {
  const char* e = std::getenv(name);
  return e && e[0] == '1';
}

int check_live(hvd_comm* c) {
  if (!c) return HVD_ERR_INVALID;
  if (c->closed) return HVD_ERR_CLOSED;
  if (*c->err_host != 0) return *c->err_host;
  if (c->size > 1 && !c->connected) return HVD_ERR_NOT_CONNECTED;
  return HVD_OK;
}

// ------------------------------------------------------------------ plan cache
void free_plan(CachedPlan& p) {
  if (p.dmem) cudaFree(p.dmem);
  if (p.hmem) cudaFreeHost(p.hmem);
  p.dmem = p.hmem = nullptr;
}

size_t align256(size_t v) { return (v + 255) / 256 * 256; }

// Free every cached plan (after the device is done with them).
void drop_plans(std::list<CachedPlan>& cache) {
  if (!cache.empty()) cudaDeviceSynchronize();
  for (CachedPlan& p : cache) free_plan(p);
  cache.clear();
}

// Build (or fetch) the device-resident pack/unpack tables of the plan of the
// tensor list `t` (n per local rank).  The key is every tensor's address,
// count and dtype plus the threshold, so repeated calls on the same gradient
// tensors (the training loop) reuse the uploaded tables.
// Host description of one fusion buffer's member table (before upload).
struct HostBuf {
  int dtype = 0;                  // buffer (wire) dtype
  int tdtype = 0;                 // tensor dtype (0: same)
  std::vector<char*> rdst;        // [nlocal * nseg] registered: successor's addresses
  uint64_t L = 0;                 // elements
  std::vector<PackSeg> segs;      // dst_off / count / vbeg per member
  std::vector<char*> src;         // [nlocal * nseg] gather addresses
  std::vector<char*> dst;         // [nlocal * nseg] scatter addresses; empty = same as src
};

// member tiles cut in half at the end of a buffer (HVD_CFG_SOLO_TAIL; -1 = one wave of
// the solo kernel: 9 resident CTAs per SM)
uint64_t solo_tail_tiles(const hvd_comm* c);

// Pipelining slices of a channel's share of a chunk (ch_el elements): K = ceil(ch_el /
// target) slices of equal size (rounded up to the quantum g), so that no runt last slice
// adds an op and a dependency wait per ring level (a 120-channel 64 MiB ring at N = 4 had
// K = 3 with a 256-byte third slice: 614 -> 530 GB/s; rounding the target down to g made
// a 48.3 MiB buffer take K = 3 instead of 2: 482 vs 566 GB/s).
void balanced_slices(uint64_t ch_el, uint64_t target_el, uint64_t g, unsigned long long* slice_el, int* K) {
  const uint64_t t = std::max<uint64_t>(1, target_el);
  const uint64_t k = std::max<uint64_t>(1, (ch_el + t - 1) / t);  // (the target unrounded: half a share is K = 2)
  uint64_t s = ((ch_el + k - 1) / k + g - 1) / g * g;
  s = std::min<uint64_t>(s, std::max<uint64_t>(ch_el, g));
  *slice_el = s;
  *K = (int)std::max<uint64_t>(1, (ch_el + s - 1) / s);
}

// solo_kernel tiles of one member of `count` elements (vel per 16 B vector)
uint64_t solo_member_tiles(uint64_t count, uint64_t vel) {
  return ((count + vel - 1) / vel + kSoloTileVecs - 1) / kSoloTileVecs;
}

CachedPlan* lookup_plan(hvd_comm* c, const std::vector<uint64_t>& key) {
  for (auto it = c->cache.begin(); it != c->cache.end(); ++it) {
    if (it->key == key) {
      c->cache.splice(c->cache.begin(), c->cache, it);
      return &c->cache.front();
    }
  }
  return nullptr;
}

// Upload the member tables of `hb` (one device allocation, one H2D copy on the
// stream) and cache them under `key` (LRU of kPlanCacheSize plans).
int upload_plan(hvd_comm* c, std::vector<uint64_t> key, const std::vector<HostBuf>& hb, cudaStream_t s,
                CachedPlan** out) {
  // layout per buffer: [segs][src][dst][tile_seg][vbeg][solo tiles]
  struct Off { size_t segs, src, dst, rdst, tiles, vbeg, stile; uint64_t nvec, ntiles, nstile; };
  std::vector<Off> offs(hb.size());
  const uint64_t tile_vecs = (uint64_t)kPackThreads * kPackVecsPerThread;
  size_t total = 0;
  for (size_t b = 0; b < hb.size(); ++b) {
    const int esz = elem_size(hb[b].dtype);
    const uint64_t vel = kPackVecBytes / esz;
    const size_t nseg = hb[b].segs.size();
    offs[b].nvec = (hb[b].L + vel - 1) / vel;
    offs[b].ntiles = (offs[b].nvec + tile_vecs - 1) / tile_vecs;
    offs[b].segs = total;
    total = align256(total + sizeof(PackSeg) * nseg);
    offs[b].src = total;
    total = align256(total + sizeof(char*) * nseg * c->nlocal);
    offs[b].dst = total;
    if (!hb[b].dst.empty()) total = align256(total + sizeof(char*) * nseg * c->nlocal);
    offs[b].rdst = total;
    if (!hb[b].rdst.empty()) total = align256(total + sizeof(char*) * nseg * c->nlocal);
    offs[b].tiles = total;
    total = align256(total + sizeof(int) * (offs[b].ntiles + 1));
    offs[b].vbeg = total;
    total = align256(total + sizeof(unsigned long long) * nseg);
    // N = 1, one local rank, same dtype: member tiles for solo_kernel
    offs[b].nstile = 0;
    if (c->size == 1 && c->nlocal == 1 && (hb[b].tdtype == 0 || hb[b].tdtype == hb[b].dtype)) {
      for (const PackSeg& sg : hb[b].segs) offs[b].nstile += solo_member_tiles(sg.count, vel);
      offs[b].nstile += std::min<uint64_t>(offs[b].nstile, solo_tail_tiles(c));  // halves of the tail
    }
    offs[b].stile = total;
    total = align256(total + sizeof(SoloTile) * offs[b].nstile);
  }
  CachedPlan p;
  p.key = std::move(key);
  if (total) {
    CK(cudaMallocHost(&p.hmem, total));
    if (cudaMalloc(&p.dmem, total) != cudaSuccess) {
      free_plan(p);
      return HVD_ERR_CUDA;
    }
  }
  char* h = static_cast<char*>(p.hmem);
  char* d = static_cast<char*>(p.dmem);
  for (size_t b = 0; b < hb.size(); ++b) {
    const HostBuf& B = hb[b];
    const int nseg = (int)B.segs.size();
    PackSeg* segs = reinterpret_cast<PackSeg*>(h + offs[b].segs);
    char** src = reinterpret_cast<char**>(h + offs[b].src);
    int* tiles = reinterpret_cast<int*>(h + offs[b].tiles);
    unsigned long long* vb = reinterpret_cast<unsigned long long*>(h + offs[b].vbeg);
    for (int j = 0; j < nseg; ++j) {
      segs[j] = B.segs[j];
      vb[j] = B.segs[j].vbeg;
    }
    std::memcpy(src, B.src.data(), sizeof(char*) * B.src.size());
    if (!B.dst.empty()) std::memcpy(h + offs[b].dst, B.dst.data(), sizeof(char*) * B.dst.size());
    if (!B.rdst.empty()) std::memcpy(h + offs[b].rdst, B.rdst.data(), sizeof(char*) * B.rdst.size());
    // tile -> member of its first vector (merge walk); last entry = last member
    int sidx = 0;
    for (uint64_t tile = 0; tile < offs[b].ntiles; ++tile) {
      const uint64_t v = tile * tile_vecs;
      while (sidx + 1 < nseg && segs[sidx + 1].vbeg <= v) ++sidx;
      tiles[tile] = sidx;
    }
    tiles[offs[b].ntiles] = nseg - 1;
    if (offs[b].nstile) {
      // member tiles: whole 16 B vectors by bulk copy (+ the ragged last elements), or, for a
      // member whose tensor is not 16 B aligned, a range of buffer vectors for the lookup path
      SoloTile* st = reinterpret_cast<SoloTile*>(h + offs[b].stile);
      const int esz = elem_size(B.dtype);
      const uint64_t vel = kPackVecBytes / esz;
      uint64_t k = 0;
      for (int j = 0; j < nseg; ++j) {
        const PackSeg& sg = B.segs[j];
        if (sg.count == 0) continue;
        const char* g = B.src[j];
        const char* dd = B.dst.empty() ? B.src[j] : B.dst[j];
        const bool mis = ((reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(dd)) & 15) != 0;
        const uint64_t nv = (sg.count + vel - 1) / vel, full = sg.count / vel;
        for (uint64_t v = 0; v < nv; v += kSoloTileVecs) {
          const uint64_t e = std::min<uint64_t>(nv, v + kSoloTileVecs);
          SoloTile& T = st[k++];
          T.member = (unsigned)j;
          if (mis) {
            T.src = sg.vbeg + v;
            T.dst = sg.vbeg + e;
            T.bytes = 0;
            T.ragged = 0;
            T.flags = 1;
          } else {
            const uint64_t fe = std::min<uint64_t>(full, e);
            T.src = reinterpret_cast<uintptr_t>(g) + v * kPackVecBytes;
            T.dst = reinterpret_cast<uintptr_t>(dd) + v * kPackVecBytes;
            T.bytes = (unsigned)((fe > v ? fe - v : 0) * kPackVecBytes);
            T.ragged = e > full ? (unsigned)(sg.count - full * vel) : 0;
            T.flags = 0;
          }
        }
      }
      // HVD_CFG_SOLO_TAIL: the last tiles are cut in half (the block scheduler runs tiles
      // in order, so the final wave drains sooner)
      const uint64_t nt = k, ns = std::min<uint64_t>(nt, offs[b].nstile - nt);
      for (uint64_t i = nt; i-- > nt - ns;) {
        const SoloTile T = st[i];
        SoloTile& a = st[i + (i - (nt - ns))];
        SoloTile& z = st[i + (i - (nt - ns)) + 1];
        const unsigned half = T.flags ? 0 : T.bytes / 32 * 16;
        a = T;
        z = T;
        if (T.flags) {  // vector range of a misaligned member
          const uint64_t mid = T.src + (T.dst - T.src) / 2;
          a.dst = mid;
          z.src = mid;
        } else {
          a.bytes = half;
          a.ragged = 0;
          z.src = T.src + half;
          z.dst = T.dst + half;
          z.bytes = T.bytes - half;
        }
      }
    }
    DevPlanBuffer db;
    db.dtype = B.dtype;
    db.tdtype = B.tdtype ? B.tdtype : B.dtype;
    db.L = B.L;
    std::memset(&db.pp, 0, sizeof(db.pp));
    db.pp.segs = reinterpret_cast<const PackSeg*>(d + offs[b].segs);
    db.pp.src = reinterpret_cast<char* const*>(d + offs[b].src);
    db.dst = B.dst.empty() ? nullptr : reinterpret_cast<char* const*>(d + offs[b].dst);
    db.rdst = B.rdst.empty() ? nullptr : reinterpret_cast<char* const*>(d + offs[b].rdst);
    db.pp.tile_seg = reinterpret_cast<const int*>(d + offs[b].tiles);
    db.vbeg = reinterpret_cast<const unsigned long long*>(d + offs[b].vbeg);
    for (int l = 0; l < c->nlocal; ++l) db.pp.buf[l] = c->rk[l].buf;
    db.pp.nvec = offs[b].nvec;
    db.pp.tile_vecs = tile_vecs;
    db.pp.ntiles = offs[b].ntiles;
    db.pp.nseg = nseg;
    db.stile = offs[b].nstile ? reinterpret_cast<const SoloTile*>(d + offs[b].stile) : nullptr;
    db.nstile = offs[b].nstile;
    for (uint64_t i = 0; i < offs[b].nstile; ++i)
      db.stile_slow |= reinterpret_cast<const SoloTile*>(h + offs[b].stile)[i].flags != 0;
    p.bufs.push_back(db);
  }
  if (total) {
    if (cudaMemcpyAsync(p.dmem, p.hmem, total, cudaMemcpyHostToDevice, s) != cudaSuccess) {
      free_plan(p);
      return HVD_ERR_CUDA;
    }
  }
  if (c->cache.size() >= kPlanCacheSize) {
    cudaStreamSynchronize(s);  // the evicted tables may still be in use on the stream
    free_plan(c->cache.back());
    c->cache.pop_back();
  }
  c->cache.push_front(std::move(p));
  *out = &c->cache.front();
  return HVD_OK;
}

// Tensor Fusion plan (hvd_plan.cpp) of the tensor list `t` (n per local rank),
// uploaded and cached by (addresses, counts, dtypes, threshold): a training loop
// that reduces the same gradient tensors every step uploads its tables once.
// dst: separate outputs (same shapes as t; nullptr: in place)
int get_plan(hvd_comm* c, const hvd_tensor* t, int n, uint64_t threshold, cudaStream_t s,
             CachedPlan** out, int wire = 0, const Registration* reg = nullptr, const hvd_tensor* dst = nullptr) {
  std::vector<uint64_t> key;
  key.reserve(7 + 4 * (size_t)n * c->nlocal);
  key.push_back(0x504c414eull);  // "PLAN"
  key.push_back((uint64_t)wire);
  key.push_back(reinterpret_cast<uint64_t>(reg));
  key.push_back(threshold);
  key.push_back((uint64_t)n);
  key.push_back((uint64_t)c->nlocal);
  key.push_back(dst ? 1 : 0);
  for (int i = 0; i < n * c->nlocal; ++i) {
    key.push_back(reinterpret_cast<uint64_t>(t[i].data));
    key.push_back(t[i].count);
    key.push_back((uint64_t)t[i].dtype);
    if (dst) key.push_back(reinterpret_cast<uint64_t>(dst[i].data));
  }
  if ((*out = lookup_plan(c, key))) return HVD_OK;
  std::vector<uint64_t> counts(n);
  std::vector<int32_t> dtypes(n);
  for (int k = 0; k < n; ++k) {
    counts[k] = t[k].count;
    dtypes[k] = wire ? wire : t[k].dtype;  // with a wire dtype the buffers hold wire elements (R14)
  }
  std::vector<hvd_plan_entry> ents;
  std::vector<hvd_plan_buffer> bufs;
  int st = build_plan(counts.data(), dtypes.data(), n, threshold, c->cap, &ents, &bufs);
  if (st != HVD_OK) return st;
  std::vector<HostBuf> hb(bufs.size());
  for (size_t b = 0; b < bufs.size(); ++b) {
    const hvd_plan_buffer& pb = bufs[b];
    const int esz = elem_size(pb.dtype);                                  // wire element size
    const int tesz = elem_size(t[ents[pb.first_entry].tensor].dtype);     // tensor element size
    const uint64_t vel = kPackVecBytes / esz;
    hb[b].dtype = pb.dtype;
    hb[b].tdtype = t[ents[pb.first_entry].tensor].dtype;
    hb[b].L = pb.length;
    hb[b].segs.resize(pb.n_entries);
    hb[b].src.resize((size_t)pb.n_entries * c->nlocal);
    for (int j = 0; j < pb.n_entries; ++j) {
      const hvd_plan_entry& e = ents[pb.first_entry + j];
      hb[b].segs[j] = {e.dst_off, e.count, e.dst_off / vel, 0};
      for (int l = 0; l < c->nlocal; ++l)
        hb[b].src[(size_t)l * pb.n_entries + j] =
            static_cast<char*>(t[(size_t)l * n + e.tensor].data) + e.src_off * tesz;
      if (dst) {
        hb[b].dst.resize((size_t)pb.n_entries * c->nlocal);
        for (int l = 0; l < c->nlocal; ++l)
          hb[b].dst[(size_t)l * pb.n_entries + j] = static_cast<char*>(dst[(size_t)l * n + e.tensor].data) + e.src_off * tesz;
      }
      if (reg) {
        hb[b].rdst.resize((size_t)pb.n_entries * c->nlocal);
        for (int l = 0; l < c->nlocal; ++l)
          hb[b].rdst[(size_t)l * pb.n_entries + j] = reg->succ[(size_t)l * n + e.tensor] + e.src_off * tesz;
      }
    }
  }
  return upload_plan(c, std::move(key), hb, s, out);
}

// ------------------------------------------------------------------ launch accounting
cudaEvent_t pool_event(hvd_comm* c) {
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Wraps one kernel launch: counts it and, when profiling, brackets it with events.
constexpr size_t kMaxTimed = 1 << 16;
// Payload bytes a launch reduces or copies (job timeline): its fusion buffers in the
// wire dtype, or the ring's one buffer.
uint64_t fused_bytes(const FusedParams& F) {
  const uint64_t esz = (uint64_t)elem_size(F.dtype);
  if (F.nbuf <= 0) return F.ring.L * esz;
  uint64_t b = 0;
  for (int i = 0; i < F.nbuf && i < kMaxMultiBufs; ++i) b += F.bufs[i].L * esz;
  return b;
}

// Issue one kernel launch: launch statistics, optional per-launch events
// (HVD_CFG_PROFILE) and the job timeline record (jt: the launch's JtRef field, filled
// in before `launch` reads the parameters).  A launcher with no work issues no kernel
// and is neither counted nor traced.
template <class F>
int launch_counted(hvd_comm* c, int kind, cudaStream_t s, JtRef* jt, uint64_t bytes, F&& launch) {
  hvd_comm::Timed t = {kind, nullptr, nullptr};
  *jt = c->jt ? c->jt->reserve() : JtRef{nullptr, nullptr, 0};
  // per-launch events until hvd_kernel_stats collects them (bounded: a caller that
  // never collects stops being profiled instead of growing without limit)
  const bool prof = c->profile && c->timed.size() < kMaxTimed;
  if (prof) {
    t.a = pool_event(c);
    t.b = pool_event(c);
    CK(cudaEventRecord(t.a, s));
  }
  const unsigned long long before = kernels_launched();
  CK(launch());
  if (kernels_launched() == before) {
    if (prof) {
      c->event_pool.push_back(t.a);
      c->event_pool.push_back(t.b);
    }
    return HVD_OK;
  }
  c->launches[kind] += 1;
  if (c->jt) c->jt->launched(kind, bytes);
  if (prof) {
    CK(cudaEventRecord(t.b, s));
    c->timed.push_back(t);
  }
  return HVD_OK;
}

// ------------------------------------------------------------------ ring enqueue
// Split one buffer of L elements for the ring kernel and launch it.
// Split one buffer of L elements into chunks / channels / slices (R2) for the
// ring or fused kernel.  Returns the channel count.
int make_ring_params(hvd_comm* c, uint64_t L, int dtype, bool fused, RingParams* P, int* nch_out,
                     uint64_t q_override = 0, bool pull = false, bool bulk = false) {
  const int esz = elem_size(dtype);
  const uint64_t g = kChunkQuantum / esz;
  std::memset(P, 0, sizeof(*P));
  for (int l = 0; l < c->nlocal; ++l) P->rk[l] = c->rk[l];
  P->N = c->size;
  P->L = L;
  P->q = q_override ? q_override : chunk_len(L, c->size, dtype);
  // channels: at least 32 KiB of every chunk per channel, at most the knob and
  // what stays co-resident (the CTAs of all ranks wait on each other)
  const int threads = pull ? std::max(256, c->threads) : c->threads;
  // occupancy of (kernel, dtype, threads), cached: a driver query per launch costs microseconds
  const int okey = bulk ? 300000000 + dtype * 10000000 + c->bulk_stages * 1000000 + (c->bulk_stage_bytes >> 10)
                       : (pull ? 2 : fused ? 1 : 0) * 100000 + dtype * 10000 + threads;
  int max_per_sm = 0;
  for (auto& kv : c->occ_cache)
    if (kv.first == okey) max_per_sm = kv.second;
  if (max_per_sm == 0) {
    CK(bulk ? bulk_max_ctas_per_sm(dtype, c->bulk_stages, c->bulk_stage_bytes, &max_per_sm)
       : pull ? pull_max_ctas_per_sm(dtype, threads, &max_per_sm)
            : fused ? fused_max_ctas_per_sm(dtype, threads, &max_per_sm) : ring_max_ctas_per_sm(dtype, threads, &max_per_sm));
    max_per_sm = std::max(1, max_per_sm);
    c->occ_cache.push_back({okey, max_per_sm});
  }
  const int resident = std::max(1, c->sm_count * max_per_sm / c->nlocal);
  const uint64_t qbytes = P->q * esz;
  int nch = (int)std::min<uint64_t>((uint64_t)(bulk ? c->bulk_channels : c->channels),
                                    std::max<uint64_t>(1, qbytes / (32 << 10)));
  nch = std::min(nch, std::min(resident, kMaxChannels));
  P->ch_el = (P->q + (uint64_t)nch * g - 1) / ((uint64_t)nch * g) * g;
  uint64_t sb = bulk ? (uint64_t)c->bulk_slice : (uint64_t)c->slice_bytes;
  if (sb == 0) sb = std::min<uint64_t>(128 << 10, std::max<uint64_t>(32 << 10, P->ch_el * esz / 2));
  balanced_slices(P->ch_el, sb / esz, g, &P->slice_el, &P->K);
  P->mode = kRingAllreduce;
  P->err = c->err_dev;
  P->timeout_ns = (unsigned long long)c->timeout_ms * 1000000ull;
  P->sig_mode = c->sig_mode;
  P->sig_warps = fused ? c->sig_warps : 1;
  P->tl = c->tl;
  P->window = c->window;
  P->fin_lag = c->fin_lag;
  P->pdl = fused ? c->fused_pdl : 0;
  P->preissue = fused ? (c->preissue < 0 ? (c->size > 2 ? 1 : 0) : c->preissue) : 0;
  P->ll_pdl = c->ll_pdl;
  // the watcher is one more warp: only while the block stays within the kernel's 416 threads
  P->watcher = fused && c->watcher && c->threads + 32 * (P->sig_warps + 1) <= kMaxRingThreads + 32 ? 1 : 0;
  if (fused && c->pace_gbps > 0 && c->size > 1) {
    // one row of remote stores = threads x 16 B; channel share of the paced rank rate
    const double row = 16.0 * c->threads;
    const double per_ch = (double)c->pace_gbps * 1e9 / nch;
    const double cyc = row / per_ch * 1e9;  // ns per row (%globaltimer)
    P->pace_cyc = (unsigned)std::max(1.0, cyc);
    P->pace_burst = (unsigned)std::min(1e9, cyc * c->pace_burst_rows);
  }
  P->tl_max = c->tl ? c->tl_max : 0;
  for (int ch = 0; ch < kMaxChannels; ++ch) P->base[ch] = pull ? c->pbase[ch] : c->base[ch];
  *nch_out = nch;
  return HVD_OK;
}

void advance_base(hvd_comm* c, const RingParams& P, int nch) {
  const unsigned long long inc = ring_signals(kRingAllreduce, c->size, P.K);
  for (int ch = 0; ch < nch; ++ch) c->base[ch] += inc;
}

// Hash of a launch's geometry: both ends of every ring link must agree on it.
struct CallHash {
  uint64_t h = 0x9e3779b97f4a7c15ull;
  void add(uint64_t v) {
    uint64_t z = (h ^ v) + 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    h = z ^ (z >> 31);
  }
};

int enqueue_ring(hvd_comm* c, uint64_t L, int dtype, cudaStream_t s) {
  if (c->size <= 1 || L == 0) return HVD_OK;
  RingParams P;
  int nch = 0;
  int st = make_ring_params(c, L, dtype, false, &P, &nch);
  if (st != HVD_OK) return st;
  P.epoch = ++c->hs_epoch;
  {
    CallHash ch;
    for (uint64_t v : {(uint64_t)1, L, (uint64_t)dtype, (uint64_t)nch, (uint64_t)P.K, (uint64_t)c->size}) ch.add(v);
    P.hash = ch.h;
  }
  st = launch_counted(c, HVD_KERNEL_RING, s, &P.jt, L * elem_size(dtype), [&] { return launch_ring(P, dtype, nch, c->nlocal, c->threads, s); });
  if (st != HVD_OK) return st;
  advance_base(c, P, nch);
  return HVD_OK;
}

// Pull protocol (pull_allreduce_kernel): ranks load their predecessor's partials.
int enqueue_pull(hvd_comm* c, DevPlanBuffer& b, cudaStream_t s) {
  FusedParams F;
  std::memset(&F, 0, sizeof(F));
  int nch = 0;
  int st = make_ring_params(c, b.L, b.dtype, true, &F.ring, &nch, 0, true);
  if (st != HVD_OK) return st;
  const int call = ++c->pull_calls;
  F.ring.call = call;
  F.ring.parity = call & 1;
  F.ring.exits_target = c->pull_exits + nch;
  F.segs = b.pp.segs;
  F.src = b.pp.src;
  F.dst = b.dst;
  F.vbeg_global = b.vbeg;
  F.nseg = b.pp.nseg;
  F.scale_on = b.pp.scale_on;
  F.scale = b.pp.scale;
  F.dtype = b.dtype;
  const int threads = std::max(256, c->threads);
  st = launch_counted(c, HVD_KERNEL_PULL, s, &F.ring.jt, fused_bytes(F), [&] { return launch_pull(F, b.dtype, nch, c->nlocal, threads, s); });
  if (st != HVD_OK) return st;
  if (c->tl) {
    c->tl_nch = nch;
    c->tl_K = F.ring.K;
    c->tl_T = 2 * c->size - 1;  // pull ops: steps 0..2N-2
    c->tl_slices = c->tl_T * F.ring.K;
    c->tl_kind = 1;
  }
  c->pull_exits += nch;
  const unsigned long long inc = (unsigned long long)(2 * c->size - 1) * F.ring.K;
  for (int ch = 0; ch < nch; ++ch) c->pbase[ch] += inc;
  return HVD_OK;
}

// One fused launch for consecutive fusion buffers of one dtype (<= kMaxMultiBufs).
// multi-buffer calls with at most this many buffers run them concurrently (disjoint
// channel ranges); with more, one channel minimum per buffer would leave the large
// buffers too few channels
constexpr int kDisjointMaxBufs = 16;

int enqueue_fused_multi(hvd_comm* c, DevPlanBuffer* const* bs, int nb, cudaStream_t s) {
  const int dtype = bs[0]->dtype;
  const int esz = elem_size(dtype);
  const uint64_t g = kChunkQuantum / esz;
  const int N = c->size;
  FusedParams F;
  std::memset(&F, 0, sizeof(F));
  // channels: sized by the largest buffer, like a single-buffer launch
  uint64_t maxL = 0;
  for (int i = 0; i < nb; ++i) maxL = std::max<uint64_t>(maxL, bs[i]->L);
  // bulk push (bulk_allreduce_kernel): same-dtype calls only (the wire conversions stay in
  // the fused kernel); the decision depends only on rank-independent call properties
  const bool bulk = c->protocol == 2 && N > 1 && bs[0]->tdtype == dtype;
  int nch = 0;
  int st = make_ring_params(c, maxL, dtype, true, &F.ring, &nch, 0, false, bulk);
  if (st != HVD_OK) return st;
  F.region_el = c->bufsz / esz / nch / g * g;
  F.bulk_stages = c->bulk_stages;
  F.bulk_stage_bytes = c->bulk_stage_bytes;
  F.bulk_depth = c->bulk_depth;
  F.scale_on = bs[0]->pp.scale_on;
  F.scale = bs[0]->pp.scale;
  F.dtype = dtype;
  F.tdtype = bs[0]->tdtype;
  F.registered = bs[0]->rdst != nullptr && N > 1;
  F.nbuf = nb;
  int maxseg = 0;
  std::vector<unsigned long long> signals(nch, 0);
  // Channels per buffer.  One buffer: all.  Several: ~64 KiB of every chunk per channel
  // (want), at least enough channels for the buffer's slots to fit their private regions
  // (need).  When every buffer's need fits, the channels are split into disjoint ranges
  // in proportion to the buffers' sizes, so all buffers of the call run at once;
  // otherwise ranges of `want` channels are assigned round robin (they overlap and a
  // channel runs its buffers in order).
  // (disjoint ranges only for a few buffers: with many, one channel minimum per buffer
  // would leave the large buffers too few channels)
  std::vector<int> kk(nb, nch), first(nb, -1);
  if (nb > 1 && nch > 1) {
    std::vector<int> want(nb), need(nb);
    std::vector<uint64_t> qs(nb);
    long sum_want = 0, sum_need = 0;
    for (int i = 0; i < nb; ++i) {
      qs[i] = chunk_len(bs[i]->L, N, dtype);
      want[i] = (int)std::min<uint64_t>((uint64_t)nch, std::max<uint64_t>(1, (qs[i] * esz + (64 << 10) - 1) / (64 << 10)));
      int k = 1;
      while (k < nch && (uint64_t)N * ((qs[i] + (uint64_t)k * g - 1) / ((uint64_t)k * g) * g) > F.region_el) ++k;
      need[i] = k;
      sum_want += want[i];
      sum_need += need[i];
    }
    if (sum_need <= nch && nb <= kDisjointMaxBufs) {
      int used = 0;
      for (int i = 0; i < nb; ++i) {
        kk[i] = sum_want <= nch ? std::max(want[i], need[i])
                                : std::max(need[i], (int)((long)nch * want[i] / sum_want));
        used += kk[i];
      }
      while (used > nch) {  // trim the buffer with the most channels above its need
        int j = -1;
        for (int i = 0; i < nb; ++i)
          if (kk[i] > need[i] && (j < 0 || kk[i] > kk[j])) j = i;
        --kk[j];
        --used;
      }
      if (sum_want > nch)
        while (used < nch) {  // spare channels to the buffer with the most data per channel
          int j = 0;
          for (int i = 1; i < nb; ++i)
            if (qs[i] * kk[j] > qs[j] * kk[i]) j = i;
          ++kk[j];
          ++used;
        }
      int f = 0;
      for (int i = 0; i < nb; ++i) {
        first[i] = kk[i] < nch ? f : -1;
        f += kk[i];
      }
    } else {
      int next_owner = 0;
      for (int i = 0; i < nb; ++i) {
        kk[i] = std::max(want[i], need[i]);
        first[i] = kk[i] < nch ? next_owner : -1;
        if (kk[i] < nch) next_owner = (next_owner + kk[i]) % nch;
      }
    }
  }
  for (int i = 0; i < nb; ++i) {
    const DevPlanBuffer& b = *bs[i];
    BufDesc& D = F.bufs[i];
    D.segs = b.pp.segs;
    D.src = b.pp.src;
    D.dst = b.dst ? b.dst : b.pp.src;
    D.rdst = b.rdst;
    D.vbeg = b.vbeg;
    D.tile_seg = b.pp.tile_seg;
    D.tile_vecs = b.pp.tile_vecs;
    D.nseg = b.pp.nseg;
    D.stile = N == 1 ? b.stile : nullptr;
    D.nstile = N == 1 ? b.nstile : 0;
    D.L = b.L;
    D.q = chunk_len(b.L, N, dtype);
    const int k = kk[i];
    D.owner = first[i];  // first channel of the range (-1: all channels)
    D.nch = k;
    D.ch_el = (D.q + (uint64_t)k * g - 1) / ((uint64_t)k * g) * g;
    uint64_t sb = bulk ? (uint64_t)c->bulk_slice : (uint64_t)c->slice_bytes;
    if (sb == 0) sb = std::min<uint64_t>(128 << 10, std::max<uint64_t>(32 << 10, D.ch_el * esz / 2));
    balanced_slices(D.ch_el, sb / esz, g, &D.slice_el, &D.K);
    if ((uint64_t)N * D.ch_el > F.region_el) return HVD_ERR_INVALID;  // region slack exhausted
    maxseg = std::max(maxseg, D.nseg);
    const unsigned long long inc = (unsigned long long)(N > 1 ? 2 * (N - 1) : 0) * D.K;
    for (int j = 0; j < k; ++j) signals[D.owner < 0 ? j : (D.owner + j) % nch] += inc;
  }
  F.cache_segs = maxseg <= kFusedSmemSegs ? (maxseg + 1) / 2 * 2 : 0;
  if (N == 1) {  // no ring: the in-place gather x (1/N) -> scatter stream
    if (c->tl) c->tl_slices = 0;  // the solo kernels record no timeline
    if (c->solo_kernel == 1 && F.tdtype == dtype) {
      // persistent bulk kernel (N = 1 branch of bulk_allreduce_kernel): every SM streams
      // tiles HBM -> shared -> HBM by bulk copies, launched with programmatic dependent
      // launch so that back-to-back calls do not pay the launch gap
      F.bulk_stages = c->solo_stages;
      F.bulk_stage_bytes = c->solo_stage_bytes;
      F.bulk_depth = 1;
      int per_sm = 0;
      CK(bulk_max_ctas_per_sm(dtype, c->solo_stages, c->solo_stage_bytes, &per_sm, false));
      const int grid = std::max(1, std::max(1, per_sm) * c->sm_count / c->nlocal);
      return launch_counted(c, HVD_KERNEL_SOLO, s, &F.ring.jt, fused_bytes(F), [&] { return launch_bulk(F, dtype, grid, c->nlocal, s); });
    }
    F.solo_tpc = 1;
    if (kSoloTPC > 1 && !F.scale_on && F.tdtype == dtype) {  // several plain member tiles per CTA
      bool plain = true;
      for (int i = 0; i < nb; ++i) plain = plain && bs[i]->stile && !bs[i]->stile_slow;
      if (plain) F.solo_tpc = kSoloTPC;
    }
    return launch_counted(c, HVD_KERNEL_SOLO, s, &F.ring.jt, fused_bytes(F), [&] { return launch_solo(F, dtype, c->nlocal, s); });
  }
  const int tdt = F.tdtype;
  F.ring.epoch = ++c->hs_epoch;
  {
    CallHash h;
    for (uint64_t v : {(uint64_t)(bulk ? 3 : 2), (uint64_t)N, (uint64_t)dtype, (uint64_t)F.tdtype,
                       (uint64_t)F.registered, (uint64_t)F.scale_on, (uint64_t)nb, (uint64_t)nch})
      h.add(v);
    for (int i = 0; i < nb; ++i)
      for (uint64_t v : {(uint64_t)F.bufs[i].L, (uint64_t)F.bufs[i].K, (uint64_t)(int64_t)F.bufs[i].owner, (uint64_t)F.bufs[i].nch})
        h.add(v);
    F.ring.hash = h.h;
  }
  if (bulk)
    st = launch_counted(c, HVD_KERNEL_BULK, s, &F.ring.jt, fused_bytes(F), [&] { return launch_bulk(F, dtype, nch, c->nlocal, s); });
  else
    st = launch_counted(c, HVD_KERNEL_FUSED, s, &F.ring.jt, fused_bytes(F), [&] { return launch_fused(F, dtype, nch, c->nlocal, c->threads, s); });
  (void)tdt;
  if (st != HVD_OK) return st;
  if (c->tl) {
    c->tl_nch = nch;
    c->tl_K = F.bufs[0].K;
    c->tl_T = N > 1 ? 2 * (N - 1) : 0;
    int ops = 0;
    for (int i = 0; i < nb; ++i)
      ops += N > 1 ? (F.registered ? c->tl_T : c->tl_T + 1) * F.bufs[i].K : F.bufs[i].K;
    c->tl_slices = ops;
    c->tl_kind = F.registered ? 2 : 0;
  }
  for (int ch = 0; ch < nch; ++ch) c->base[ch] += signals[ch];
  return HVD_OK;
}

// LL protocol (ll_allreduce_kernel) for a group of small buffers of one dtype in
// one cooperative launch: buffer i gets nch_i CTAs (one 16 B vector per thread per
// step where the co-resident budget allows) and its own slot area in each parity half.
int ll_want(const hvd_comm* c, const DevPlanBuffer& b, uint64_t cta_bytes) {
  const uint64_t q = chunk_len(b.L, c->size, b.dtype);
  const uint64_t qb = q * elem_size(b.dtype);
  return (int)std::min<uint64_t>((uint64_t)c->ll_ctas, std::max<uint64_t>(1, (qb + cta_bytes - 1) / cta_bytes));
}

// cta_bytes: chunk bytes per CTA (4 KiB = one 16 B vector per thread per step for a lone
// buffer; 16 KiB when many buffers share the launch)
int enqueue_ll(hvd_comm* c, DevPlanBuffer* const* bs, int nb, cudaStream_t s, uint64_t cta_bytes = 4096) {
  const int dtype = bs[0]->dtype;
  const int esz = elem_size(dtype);
  const uint64_t g = kChunkQuantum / esz;
  const int N = c->size;
  FusedParams F;
  std::memset(&F, 0, sizeof(F));
  int nch_unused = 0;
  int st = make_ring_params(c, bs[0]->L, dtype, true, &F.ring, &nch_unused);
  if (st != HVD_OK) return st;
  int ctas = 0;
  uint64_t words = 0;
  for (int i = 0; i < nb; ++i) {
    const DevPlanBuffer& b = *bs[i];
    BufDesc& D = F.bufs[i];
    D.q = chunk_len(b.L, N, dtype);
    D.nch = ll_want(c, b, cta_bytes);
    ctas += D.nch;
    D.segs = b.pp.segs;
    D.src = b.pp.src;
    D.dst = b.dst ? b.dst : b.pp.src;
    D.vbeg = b.vbeg;
    D.tile_seg = b.pp.tile_seg;
    D.tile_vecs = b.pp.tile_vecs;
    D.nseg = b.pp.nseg;
    D.L = b.L;
    D.ch_el = (D.q + (uint64_t)D.nch * g - 1) / ((uint64_t)D.nch * g) * g;
    D.slice_el = std::max<uint64_t>(D.ch_el, g);
    D.K = 1;
    D.owner = -1;
    D.ll_off = (unsigned)words;
    words += (uint64_t)2 * (N - 1) * (D.q * esz / 16 * 4);  // T steps x slot (8 B word per 4 B of data)
  }
  if (ctas > c->ll_ctas || words * 8 > kLLHalfBytes) return HVD_ERR_INVALID;
  F.nbuf = nb;
  F.scale_on = bs[0]->pp.scale_on;
  F.scale = bs[0]->pp.scale;
  F.dtype = dtype;
  F.tdtype = dtype;
  F.ring.epoch = ++c->ll_epoch;
  if (c->tl) c->tl_slices = 0;  // the LL kernel records no timeline
  return launch_counted(c, HVD_KERNEL_LL, s, &F.ring.jt, fused_bytes(F), [&] { return launch_ll(F, dtype, ctas, c->nlocal, s); });
}

// LL for a lone buffer up to ll_max; inside a multi-buffer plan only for buffers of at
// most kLLMultiBytes (larger ones pipeline better inside the multi-buffer fused launch)
// (measured on Inception V3 with fusion off, profiles/r01_ll_multi_limit.json: at N = 2
// 256 KiB is best; at N = 4 1 MiB cuts bf16 from 679 to 413 us and fp32 from 686 to 649 us)
constexpr int64_t kLLMultiBytes = 256 << 10;     // N = 2
constexpr int64_t kLLMultiBytesN4 = 1 << 20;     // N > 2
// LL128 (ll128_allreduce_kernel) for one buffer: pairs of 128-byte lines carrying 15
// vectors and two 8-byte flags.
uint64_t ll128_lines(const hvd_comm* c, const DevPlanBuffer& b) {
  const uint64_t qv = chunk_len(b.L, c->size, b.dtype) * elem_size(b.dtype) / 16;
  return 2 * ((qv + 14) / 15);
}

bool ll128_eligible(const hvd_comm* c, const DevPlanBuffer& b) {
  const int64_t bytes = (int64_t)(b.L * elem_size(b.dtype));
  return c->size > 1 && c->protocol >= 1 && b.L > 0 && b.tdtype == b.dtype && b.dtype != HVD_INT64 &&
         bytes > c->ll_max && bytes <= c->ll128_max &&
         (uint64_t)2 * (c->size - 1) * ll128_lines(c, b) * 128 <= kLL128HalfBytes;  // fits a half
}

int ll128_want(const hvd_comm* c, const DevPlanBuffer& b, uint64_t lines_per_cta = 32) {
  // lone buffer: one group of 4 lines per warp per step where the co-resident budget
  // allows (8 warps, 32 lines); in a group of buffers, 4 groups per warp (128 lines)
  return (int)std::min<uint64_t>((uint64_t)c->ll_ctas,
                                 std::max<uint64_t>(1, (ll128_lines(c, b) + lines_per_cta - 1) / lines_per_cta));
}
uint64_t ll128_words(const hvd_comm* c, const DevPlanBuffer& b) {
  return (uint64_t)2 * (c->size - 1) * ll128_lines(c, b) * 16;
}

// A group of buffers of one dtype in one LL128 launch: buffer i gets its own CTAs and
// its own slot area in the launch's half.
int enqueue_ll128(hvd_comm* c, DevPlanBuffer* const* bs, int nb, cudaStream_t s) {
  const int dtype = bs[0]->dtype;
  FusedParams F;
  std::memset(&F, 0, sizeof(F));
  int nch_unused = 0;
  int st = make_ring_params(c, bs[0]->L, dtype, true, &F.ring, &nch_unused);
  if (st != HVD_OK) return st;
  int ctas = 0;
  uint64_t words = 0;
  for (int i = 0; i < nb; ++i) {
    const DevPlanBuffer& b = *bs[i];
    BufDesc& D = F.bufs[i];
    D.q = chunk_len(b.L, c->size, dtype);
    D.segs = b.pp.segs;
    D.src = b.pp.src;
    D.dst = b.dst ? b.dst : b.pp.src;
    D.vbeg = b.vbeg;
    D.tile_seg = b.pp.tile_seg;
    D.tile_vecs = b.pp.tile_vecs;
    D.nseg = b.pp.nseg;
    D.L = b.L;
    D.ch_el = D.q;
    D.slice_el = D.q;
    D.K = 1;
    D.owner = -1;
    D.nch = ll128_want(c, b, nb > 1 ? 128 : 32);
    D.ll_off = (unsigned)words;
    ctas += D.nch;
    words += ll128_words(c, b);
  }
  if (ctas > c->ll_ctas || words * 8 > kLL128HalfBytes) return HVD_ERR_INVALID;
  F.nbuf = nb;
  F.scale_on = bs[0]->pp.scale_on;
  F.scale = bs[0]->pp.scale;
  F.dtype = dtype;
  F.tdtype = dtype;
  // one epoch sequence for LL and LL128 launches; each protocol alternates the two halves
  // of its own area, so a half is reused at least two launches later (after the ring's
  // dependency chain of the launch in between)
  F.ring.epoch = ++c->ll_epoch;
  if (c->tl) c->tl_slices = 0;
  return launch_counted(c, HVD_KERNEL_LL128, s, &F.ring.jt, fused_bytes(F), [&] { return launch_ll128(F, dtype, ctas, c->nlocal, s); });
}

bool ll_eligible(const hvd_comm* c, const DevPlanBuffer& b, bool multi) {
  const int esz = elem_size(b.dtype);
  // (ll_max == 0 turns LL off everywhere; otherwise multi-buffer calls have their own limit)
  const int64_t lim = c->ll_max == 0 ? 0 : multi ? (c->size <= 2 ? kLLMultiBytes : kLLMultiBytesN4) : c->ll_max;
  return c->size > 1 && c->protocol >= 1 && b.L > 0 && b.tdtype == b.dtype && b.dtype != HVD_INT64 &&
         (int64_t)(b.L * esz) <= lim;
}

// The fused path for a whole plan: small buffers through the LL protocol (grouped),
// the rest through multi-buffer fused launches (or the pull protocol per buffer).
int enqueue_fused_plan(hvd_comm* c, CachedPlan* plan, cudaStream_t s) {
  if (plan->bufs.size() == 1 && ll128_eligible(c, plan->bufs[0])) {
    DevPlanBuffer* b0 = &plan->bufs[0];
    return enqueue_ll128(c, &b0, 1, s);
  }
  std::vector<DevPlanBuffer*> group;
  const bool multi = plan->bufs.size() > 1;
  // many buffers (fusion off) at N > 2: the mid-size ones (above the LL limit, <= 16 MiB)
  // go to grouped LL128 launches; with few buffers they run concurrently in the fused
  // launch, and at N = 2 the fused ring's two steps are short enough
  const bool many = (int)plan->bufs.size() > kDisjointMaxBufs;
  auto ll128_multi = [&](const DevPlanBuffer& b) {
    return many && !ll_eligible(c, b, multi) && c->ll128_max > 0 && c->size > 2 && c->protocol >= 1 && b.L > 0 &&
           b.tdtype == b.dtype && b.dtype != HVD_INT64 &&
           (int64_t)(b.L * elem_size(b.dtype)) <= std::min<int64_t>(c->ll128_max, 16ll << 20) &&
           ll128_words(c, b) * 8 <= kLL128HalfBytes;
  };
  // A few-buffer plan with a buffer for the fused launch: its small buffers of the same
  // dtypes join that launch on channels of their own, hidden behind the large buffer,
  // instead of an LL launch serialised before it (a 64 MiB buffer + a 0.25 MiB tail at
  // N = 4: 194 -> 166 us; profiles/r02_tail_buffer/)
  bool join[8] = {};
  if (multi && !many)
    for (const DevPlanBuffer& b : plan->bufs)
      if (b.L > 0 && !ll_eligible(c, b, multi) && !ll128_multi(b) && b.tdtype == b.dtype && b.dtype >= 0 && b.dtype < 8)
        join[b.dtype] = true;
  auto small_ll = [&](const DevPlanBuffer& b) {
    return ll_eligible(c, b, multi) && !(b.dtype >= 0 && b.dtype < 8 && join[b.dtype]);
  };
  const uint64_t cta_bytes = multi ? (16 << 10) : 4096;
  // 1. LL groups: same dtype, <= kMaxMultiBufs buffers, CTA and region budgets
  {
    int ctas = 0;
    uint64_t words = 0;
    auto flush = [&]() -> int {
      int st = HVD_OK;
      if (!group.empty()) st = enqueue_ll(c, group.data(), (int)group.size(), s, cta_bytes);
      group.clear();
      ctas = 0;
      words = 0;
      return st;
    };
    for (DevPlanBuffer& b : plan->bufs) {
      if (!small_ll(b)) continue;
      const int esz = elem_size(b.dtype);
      const uint64_t q = chunk_len(b.L, c->size, b.dtype);
      const int want = ll_want(c, b, cta_bytes);
      const uint64_t w = (uint64_t)2 * (c->size - 1) * (q * esz / 16 * 4);
      if (!group.empty() && (group[0]->dtype != b.dtype || (int)group.size() >= kMaxMultiBufs ||
                             ctas + want > c->ll_ctas || (words + w) * 8 > kLLHalfBytes)) {
        int st = flush();
        if (st != HVD_OK) return st;
      }
      group.push_back(&b);
      ctas += want;
      words += w;
    }
    int st = flush();
    if (st != HVD_OK) return st;
  }
  // 1b. LL128 groups (fusion off): same dtype, <= kMaxMultiBufs, CTA and region budgets
  {
    int ctas = 0;
    uint64_t words = 0;
    auto flush = [&]() -> int {
      int st = HVD_OK;
      if (!group.empty()) st = enqueue_ll128(c, group.data(), (int)group.size(), s);
      group.clear();
      ctas = 0;
      words = 0;
      return st;
    };
    for (DevPlanBuffer& b : plan->bufs) {
      if (!ll128_multi(b)) continue;
      const int want = ll128_want(c, b, 128);
      const uint64_t w = ll128_words(c, b);
      if (!group.empty() && (group[0]->dtype != b.dtype || (int)group.size() >= kMaxMultiBufs ||
                             ctas + want > c->ll_ctas || (words + w) * 8 > kLL128HalfBytes)) {
        int st = flush();
        if (st != HVD_OK) return st;
      }
      group.push_back(&b);
      ctas += want;
      words += w;
    }
    int st = flush();
    if (st != HVD_OK) return st;
  }
  // 2. everything else
  auto flush = [&]() -> int {
    int st = HVD_OK;
    if (!group.empty()) st = enqueue_fused_multi(c, group.data(), (int)group.size(), s);
    group.clear();
    return st;
  };
  for (DevPlanBuffer& b : plan->bufs) {
    if (b.L == 0 || small_ll(b) || ll128_multi(b)) continue;
    if (c->protocol == 0 && c->pull_ok && c->size > 1 && b.tdtype == b.dtype && !b.rdst) {
      int st = flush();
      if (st != HVD_OK) return st;
      st = enqueue_pull(c, b, s);
      if (st != HVD_OK) return st;
      continue;
    }
    if (!group.empty() && (group[0]->dtype != b.dtype || group[0]->tdtype != b.tdtype ||
                           (int)group.size() >= std::min(c->multi_bufs, kMaxMultiBufs))) {
      int st = flush();
      if (st != HVD_OK) return st;
    }
    group.push_back(&b);
  }
  return flush();
}

int pack_grid(hvd_comm* c) { return c->sm_count * c->pack_ctas_per_sm / c->nlocal + 1; }

// Job timeline host span of one public call (a no-op when the timeline is off).
template <class Fn>
int traced(hvd_comm* c, const char* name, uint64_t tensors, uint64_t bytes, Fn&& fn) {
  if (!c || c->closed || !c->jt) return fn();
  c->jt->call_begin(name, tensors, bytes);
  const int st = fn();
  if (c->jt) c->jt->call_end(st);
  return st;
}
uint64_t list_bytes(const hvd_tensor* t, int n) {
  uint64_t b = 0;
  for (int k = 0; t && k < n; ++k) b += t[k].count * (uint64_t)elem_size(t[k].dtype);
  return b;
}

int do_allreduce(hvd_comm* c, const hvd_tensor* t, int n, int op, uint64_t threshold, cudaStream_t s,
                 int wire = 0, const Registration* reg = nullptr, const hvd_tensor* dst = nullptr) {
  int st = check_live(c);
  if (st != HVD_OK) return st;
  if (n < 0 || (n > 0 && !t)) return HVD_ERR_INVALID;
  if (op != HVD_SUM && op != HVD_AVERAGE) return HVD_ERR_INVALID;
  if (wire) {  // R14: one float tensor dtype, a different float wire dtype, fused kernel only
    if (wire != HVD_FLOAT32 && wire != HVD_BFLOAT16) return HVD_ERR_UNSUPPORTED;
    bool same = true;
    for (int k = 0; k < n; ++k) same = same && t[k].dtype == wire;
    if (same) {
      wire = 0;
    } else {
      for (int k = 0; k < n; ++k)
        if (t[k].dtype != t[0].dtype || (t[k].dtype != HVD_FLOAT32 && t[k].dtype != HVD_BFLOAT16))
          return HVD_ERR_UNSUPPORTED;
      if (!c->fused) return HVD_ERR_UNSUPPORTED;
    }
  }
  for (int k = 0; k < n; ++k) {
    if (elem_size(t[k].dtype) == 0) return HVD_ERR_UNSUPPORTED;
    if (op == HVD_AVERAGE && (t[k].dtype == HVD_INT32 || t[k].dtype == HVD_INT64)) return HVD_ERR_UNSUPPORTED;
    for (int l = 0; l < c->nlocal; ++l) {
      const hvd_tensor& x = t[(size_t)l * n + k];
      if (x.count != t[k].count || x.dtype != t[k].dtype) return HVD_ERR_INVALID;
      if (x.count && !x.data) return HVD_ERR_INVALID;
    }
  }
  if (n == 0) return HVD_OK;
  CK(cudaSetDevice(c->device));
  CachedPlan* plan = nullptr;
  if ((reg || dst) && !c->fused) return HVD_ERR_UNSUPPORTED;
  st = get_plan(c, t, n, threshold, s, &plan, wire, reg, dst);
  if (st != HVD_OK) return st;
  const float scale = 1.0f / (float)c->size;  // s = fl32(1/N) (R1)
  for (DevPlanBuffer& b : plan->bufs) {
    b.pp.scale = scale;
    // N = 1: s = fl32(1/1) = 1 and fl32(x * 1) = x for every x (NaN stays NaN), so the
    // prescale is the identity and is not computed (R1)
    b.pp.scale_on = op == HVD_AVERAGE && c->size > 1 ? 1 : 0;
  }
  if (c->fused) return enqueue_fused_plan(c, plan, s);  // steps 3-6, zero-copy, few launches
  for (DevPlanBuffer& b : plan->bufs) {       // step 6: repeat per fusion buffer
    PackParams pp = b.pp;
    st = launch_counted(c, HVD_KERNEL_PACK, s, &pp.jt, b.L * elem_size(b.dtype), [&] {  // step 3
      return launch_pack(pp, b.dtype, c->nlocal, pack_grid(c), kPackThreads, s);
    });
    if (st != HVD_OK) return st;
    st = enqueue_ring(c, b.L, b.dtype, s);                                    // step 4
    if (st != HVD_OK) return st;
    st = launch_counted(c, HVD_KERNEL_UNPACK, s, &pp.jt, b.L * elem_size(b.dtype), [&] {  // step 5
      return launch_unpack(pp, b.dtype, c->nlocal, pack_grid(c), kPackThreads, s);
    });
    if (st != HVD_OK) return st;
  }
  return HVD_OK;
}

// NVLink P2P status of two GPUs by PCI bus id through NVML (dlopen: no link-time
// dependency): 1 NVLink, 0 not NVLink, -1 unknown (NVML missing or the query failed).
int nvlink_link(const char* a, const char* b) {
  typedef int (*InitFn)();
  typedef int (*HandleFn)(const char*, void**);
  typedef int (*P2PFn)(void*, void*, int, int*);
  const char* chk = std::getenv("HVD_NVLINK_CHECK");  // "0": skip NVML (unknown -> LL128 off)
  if (chk && chk[0] == '0') return -1;
  static void* lib = dlopen("libnvidia-ml.so.1", RTLD_NOW | RTLD_LOCAL);
  if (!lib) return -1;
  static InitFn init = reinterpret_cast<InitFn>(dlsym(lib, "nvmlInit_v2"));
  static HandleFn handle = reinterpret_cast<HandleFn>(dlsym(lib, "nvmlDeviceGetHandleByPciBusId_v2"));
  static P2PFn p2p = reinterpret_cast<P2PFn>(dlsym(lib, "nvmlDeviceGetP2PStatus"));
  static int init_rc = init ? init() : -1;
  if (init_rc != 0 || !handle || !p2p) return -1;
  void* da = nullptr;
  void* db = nullptr;
  if (handle(a, &da) != 0 || handle(b, &db) != 0) return -1;
  if (da == db) return 1;  // one GPU (a ring of two ranks on one device is not a real comm)
  int st = -1;
  if (p2p(da, db, 2 /* NVML_P2P_CAPS_INDEX_NVLINK */, &st) != 0) return -1;
  return st == 0 /* NVML_P2P_STATUS_OK */ ? 1 : 0;
}

// The LL128 line-atomicity self-test (ll128_selftest_kernel) and the agreement on its
// outcome: every rank's count of torn or missing lines (plus `no_nvlink`, `force_fail`)
// is summed by a one-element LL allreduce — the LL protocol's 8-byte words are
// single-copy atomic by PTX, so the agreement does not depend on what is being tested.
// A non-zero sum disables LL128 on every rank (HVD_CFG_LL128_MAX_BYTES = 0).
int ll128_selftest(hvd_comm* c, int no_nvlink, int force_fail, int* status) {
  *status = 0;
  if (c->size <= 1) return HVD_OK;
  CK(cudaSetDevice(c->device));
  CK(cudaDeviceSynchronize());  // no earlier launch of this rank still reads its LL128 area
  cudaStream_t s = nullptr;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  unsigned long long* torn = nullptr;
  int st = cuda_fail(cudaMalloc(reinterpret_cast<void**>(&torn), 8 * kMaxLocal + 16 * kMaxLocal), "cudaMalloc");
  unsigned long long host[kMaxLocal] = {};
  int flag[kMaxLocal * 4] = {};  // per local rank: {torn or missing lines, not NVLink, forced, 0}
  if (st == HVD_OK) st = cuda_fail(cudaMemsetAsync(torn, 0, 8 * kMaxLocal, s), "cudaMemsetAsync");
  if (st == HVD_OK) {
    RingParams P;
    std::memset(&P, 0, sizeof(P));
    for (int l = 0; l < c->nlocal; ++l) P.rk[l] = c->rk[l];
    P.N = c->size;
    P.timeout_ns = (unsigned long long)c->timeout_ms * 1000000ull;
    P.err = c->err_dev;
    P.epoch = ++c->hs_epoch;  // the launch handshake's epoch sequence (every rank calls this)
    const int nch = std::max(1, std::min(64, c->sm_count * 2 / c->nlocal));
    st = cuda_fail(launch_ll128_selftest(P, nch, c->nlocal, 8, 256, torn, s), "ll128 self-test");
  }
  if (st == HVD_OK) st = cuda_fail(cudaMemcpyAsync(host, torn, 8 * c->nlocal, cudaMemcpyDeviceToHost, s), "copy");
  if (st == HVD_OK) st = cuda_fail(cudaStreamSynchronize(s), "self-test sync");
  int* dflag = reinterpret_cast<int*>(torn + kMaxLocal);
  if (st == HVD_OK) {
    for (int l = 0; l < c->nlocal; ++l) {
      flag[4 * l + 0] = host[l] ? 1 : 0;
      flag[4 * l + 1] = no_nvlink ? 1 : 0;
      flag[4 * l + 2] = force_fail ? 1 : 0;
      flag[4 * l + 3] = 0;
    }
    st = cuda_fail(cudaMemcpyAsync(dflag, flag, 16 * c->nlocal, cudaMemcpyHostToDevice, s), "copy");
  }
  if (st == HVD_OK) {
    std::vector<hvd_tensor> t(c->nlocal);
    for (int l = 0; l < c->nlocal; ++l) t[l] = {dflag + 4 * l, 4, HVD_INT32, 0};
    st = do_allreduce(c, t.data(), 1, HVD_SUM, c->cap, s);
  }
  if (st == HVD_OK) st = cuda_fail(cudaMemcpyAsync(flag, dflag, 16, cudaMemcpyDeviceToHost, s), "copy");
  if (st == HVD_OK) st = cuda_fail(cudaStreamSynchronize(s), "agreement sync");
  if (torn) cudaFree(torn);
  cudaStreamDestroy(s);
  if (st != HVD_OK) return st;
  // summed over the ranks: {ranks that saw torn or missing lines, ranks with a non-NVLink
  // ring link, ranks forcing a failure} — identical on every rank
  if (flag[0] == 0 && flag[1] == 0 && flag[2] == 0) {
    *status = 1;
  } else {
    *status = flag[2] ? -3 : (flag[1] ? -2 : -1);
    c->ll128_max = 0;
  }
  c->ll128_status = *status;
  return HVD_OK;
}

}  // namespace

// ================================================================== C ABI
extern "C" {

static int allreduce_host_impl(hvd_comm* c, const void* const* in, void* const* out, uint64_t count, int dtype, int op,
                               uint64_t chunk_bytes, void* stream);
static int allreduce_negotiated_impl(hvd_comm* c, hvd_negotiator* g, const hvd_tensor* tensors, uint32_t n, int op,
                                     uint64_t fusion_threshold, void* stream, uint32_t* ids_out, uint32_t* n_out);
static int allreduce_buffer_impl(hvd_comm* c, uint64_t count, int dtype, int op, void* stream);
static int broadcast_impl(hvd_comm* c, const hvd_tensor* t, int n, int root, void* stream);
static int allgather_impl(hvd_comm* c, const hvd_tensor* in, const hvd_tensor* out, void* stream);

// HVD_TIMELINE=<path> ("a single environment variable"): the job timeline of
// every comm of the process goes to <path>.  The first comm of the process that writes
// it starts a new file (rank 0 of a multi-process job: at hvd_init, before any rank can
// connect); every rank appends from then on.
static bool g_timeline_truncated = false;
static const char* timeline_env() {
  const char* p = std::getenv("HVD_TIMELINE");
  return p && p[0] ? p : nullptr;
}
static int timeline_start(hvd_comm* c, const char* path, bool truncate) {
  int ranks[kMaxLocal];
  for (int l = 0; l < c->nlocal; ++l) ranks[l] = c->rk[l].rank;
  return JobTrace::create(path, truncate, c->device, c->nlocal, ranks, c->size, &c->jt);
}
static int timeline_env_start(hvd_comm* c) {
  const char* p = timeline_env();
  if (!p || c->jt) return HVD_OK;
  const bool trunc = !g_timeline_truncated && c->rank == 0;
  g_timeline_truncated = true;
  return timeline_start(c, p, trunc);
}

int hvd_init(int rank, int size, int device, uint64_t fusion_bytes, hvd_comm** out) {
  if (!out || size < 1 || rank < 0 || rank >= size || device < 0) return HVD_ERR_INVALID;
  *out = nullptr;
  hvd_comm* c = new hvd_comm();
  c->rank = rank;
  c->size = size;
  c->device = device;
  c->nlocal = 1;
  c->virt = false;
  c->want_pull = env_on("HVD_PULL_BUFFERS");
  int st = common_init(c, fusion_bytes);
  if (st != HVD_OK) {
    hvd_finalize(c);
    return st;
  }
  if (size == 1) {
    set_neighbours(c->rk[0], c->region[0], c->region[0], c->bufsz);
    c->connected = true;
    st = timeline_env_start(c);
  } else if (rank == 0 && timeline_env() && !g_timeline_truncated) {
    // new file before any rank connects (the others append from hvd_connect on)
    FILE* f = std::fopen(timeline_env(), "w");
    if (f) {
      std::fputs("[\n", f);
      std::fclose(f);
    }
    g_timeline_truncated = true;
  }
  if (st != HVD_OK) {
    hvd_finalize(c);
    return st;
  }
  *out = c;
  return HVD_OK;
}

int hvd_init_virtual(int size, int device, uint64_t fusion_bytes, hvd_comm** out) {
  if (!out || size < 1 || size > kMaxLocal || device < 0) return HVD_ERR_INVALID;
  *out = nullptr;
  hvd_comm* c = new hvd_comm();
  c->rank = 0;
  c->size = size;
  c->device = device;
  c->nlocal = size;
  c->virt = true;
  int st = common_init(c, fusion_bytes);
  if (st != HVD_OK) {
    hvd_finalize(c);
    return st;
  }
  for (int l = 0; l < size; ++l)
    set_neighbours(c->rk[l], c->region[(l + 1) % size], c->region[(l + size - 1) % size], c->bufsz);
  c->connected = true;
  st = env_on("HVD_PULL_BUFFERS") ? alloc_pull(c) : HVD_OK;
  if (st == HVD_OK) st = timeline_env_start(c);
  if (st != HVD_OK) {
    hvd_finalize(c);
    return st;
  }
  *out = c;
  return HVD_OK;
}

int hvd_get_ipc_blob(hvd_comm* c, void* out, uint64_t* len) {
  if (!c || !len) return HVD_ERR_INVALID;
  if (c->closed) return HVD_ERR_CLOSED;
  if (!out) {
    *len = sizeof(Blob);
    return HVD_OK;
  }
  if (*len < sizeof(Blob) || c->virt) return HVD_ERR_INVALID;
  Blob b;
  std::memset(&b, 0, sizeof(b));
  b.magic = kBlobMagic;
  b.version = HVD_ABI_VERSION;
  b.rank = c->rank;
  b.size = c->size;
  b.device = c->device;
  b.pid = (int32_t)getpid();
  b.capacity = c->cap;
  b.region_bytes = kNumBufs * c->bufsz + kTailBytes + kLLRegionBytes;
  b.region_addr = reinterpret_cast<uint64_t>(c->region[0]);
  CK(cudaSetDevice(c->device));
  CK(cudaIpcGetMemHandle(&b.handle, c->region[0]));
  if (c->want_pull) {
    const int st = alloc_pull(c);
    if (st != HVD_OK) return st;
    b.has_pull = 1;
    b.pull_addr = reinterpret_cast<uint64_t>(c->pull_mem[0]);
    CK(cudaIpcGetMemHandle(&b.pull_handle, c->pull_mem[0]));
  }
  c->blob_out = true;
  CK(cudaDeviceGetPCIBusId(b.pci, (int)sizeof(b.pci), c->device));
  std::memcpy(out, &b, sizeof(b));
  *len = sizeof(Blob);
  return HVD_OK;
}

int hvd_connect(hvd_comm* c, const void* blobs, uint64_t len_each) {
  if (!c || !blobs || len_each < sizeof(Blob)) return HVD_ERR_INVALID;
  if (c->closed) return HVD_ERR_CLOSED;
  if (c->virt || c->size == 1) return HVD_OK;
  const char* p = static_cast<const char*>(blobs);
  int npull = 0;
  for (int r = 0; r < c->size; ++r) {
    Blob b;
    std::memcpy(&b, p + (size_t)r * len_each, sizeof(b));
    if (b.magic != kBlobMagic || b.version != HVD_ABI_VERSION || b.rank != r || b.size != c->size ||
        b.capacity != c->cap)
      return HVD_ERR_INVALID;
    npull += b.has_pull != 0;
  }
  // HVD_CFG_PULL_BUFFERS must be identical on every rank
  if (npull != 0 && npull != c->size) return HVD_ERR_INVALID;
  CK(cudaSetDevice(c->device));
  const int succ = (c->rank + 1) % c->size;
  const int pred = (c->rank + c->size - 1) % c->size;
  Blob bs, bp;
  std::memcpy(&bs, p + (size_t)succ * len_each, sizeof(bs));
  std::memcpy(&bp, p + (size_t)pred * len_each, sizeof(bp));
  // a peer in another process: CUDA IPC; in this process (one process driving several
  // GPUs, e.g. for profiling): its allocation directly, through peer access
  const int me_pid = (int)getpid();
  auto map_peer = [&](const Blob& b, char** out, bool* ipc) -> int {
    if (b.pid == me_pid) {
      if (b.device != c->device) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else CK(e);
      }
      *out = reinterpret_cast<char*>(b.region_addr);
      *ipc = false;
      return HVD_OK;
    }
    void* ptr = nullptr;
    CK(cudaIpcOpenMemHandle(&ptr, b.handle, cudaIpcMemLazyEnablePeerAccess));
    *out = static_cast<char*>(ptr);
    *ipc = true;
    return HVD_OK;
  };
  int mst = map_peer(bs, &c->peer_region, &c->peer_ipc);
  if (mst != HVD_OK) return mst;
  c->succ_device = bs.device;
  if (pred != succ) {
    mst = map_peer(bp, &c->pred_region, &c->pred_ipc);
    if (mst != HVD_OK) return mst;
  } else {
    c->pred_region = c->peer_region;
  }
  set_neighbours(c->rk[0], c->peer_region, c->pred_region, c->bufsz);
  if (npull == c->size) {
    if (bp.pid == me_pid) {
      c->pred_pull = reinterpret_cast<const char*>(bp.pull_addr);
    } else {
      void* ptr = nullptr;
      CK(cudaIpcOpenMemHandle(&ptr, bp.pull_handle, cudaIpcMemLazyEnablePeerAccess));
      c->pred_pull = static_cast<const char*>(ptr);
      c->pred_pull_ipc = true;
    }
    c->rk[0].ppull[0] = c->pred_pull;
    c->rk[0].ppull[1] = c->pred_pull + c->bufsz;
    c->pull_ok = true;
  }
  c->connected = true;
  // LL128 only over verified NVLink ring links whose 128-byte lines arrive whole
  // (ADVICE r1): NVML's NVLink P2P status of both links, then the line-atomicity
  // self-test; every rank applies the same agreed outcome.
  char me_pci[32] = {};
  CK(cudaDeviceGetPCIBusId(me_pci, (int)sizeof(me_pci), c->device));
  const int nv = nvlink_link(me_pci, bs.pci) == 1 && nvlink_link(me_pci, bp.pci) == 1;
  const char* ff = std::getenv("HVD_LL128_SELFTEST_FORCE_FAIL");
  int status = 0;
  const int st = ll128_selftest(c, !nv, ff && ff[0] == '1', &status);
  if (st != HVD_OK) return st;
  return timeline_env_start(c);
}

int hvd_ll128_selftest(hvd_comm* c, int force_fail, int* status) {
  int st = check_live(c);
  if (st != HVD_OK) return st;
  if (!status) return HVD_ERR_INVALID;
  return ll128_selftest(c, 0, force_fail, status);
}

int hvd_finalize(hvd_comm* c) {
  if (!c) return HVD_OK;
  if (!c->closed) {
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    if (c->jt) {  // the device is synchronised: every launch's record is final
      c->jt->drain(true);
      delete c->jt;
      c->jt = nullptr;
    }
    for (auto& p : c->cache) free_plan(p);
    for (auto& t : c->timed) {
      cudaEventDestroy(t.a);
      cudaEventDestroy(t.b);
    }
    for (auto e : c->event_pool) cudaEventDestroy(e);
    for (int k = 0; k < hvd_comm::kHostSlots; ++k) {
      if (c->ev_in[k]) cudaEventDestroy(c->ev_in[k]);
      if (c->ev_red[k]) cudaEventDestroy(c->ev_red[k]);
      if (c->ev_out[k]) cudaEventDestroy(c->ev_out[k]);
    }
    if (c->ev_start) cudaEventDestroy(c->ev_start);
    if (c->ev_done) cudaEventDestroy(c->ev_done);
    if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
    if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
    for (int l = 0; l < kMaxLocal; ++l)
      if (c->stage[l]) cudaFree(c->stage[l]);
    drop_plans(c->cache);
    for (auto& kv : c->ipc_maps) cudaIpcCloseMemHandle(kv.second);
    if (c->peer_region && c->peer_ipc) cudaIpcCloseMemHandle(c->peer_region);
    if (c->pred_region && c->pred_region != c->peer_region && c->pred_ipc) cudaIpcCloseMemHandle(c->pred_region);
    if (c->pred_pull && c->pred_pull_ipc) cudaIpcCloseMemHandle(const_cast<char*>(c->pred_pull));
    for (int l = 0; l < kMaxLocal; ++l) {
      if (c->region[l]) cudaFree(c->region[l]);
      if (c->pull_mem[l]) cudaFree(c->pull_mem[l]);
    }
    if (c->err_host) cudaFreeHost(c->err_host);
    if (c->err_dev) cudaFree(c->err_dev);
    if (c->tl) cudaFree(c->tl);
    c->closed = true;
  }
  delete c;
  return HVD_OK;
}

int hvd_rank(const hvd_comm* c) { return c ? c->rank : -1; }
int hvd_size(const hvd_comm* c) { return c ? c->size : -1; }
int hvd_local_ranks(const hvd_comm* c) { return c ? c->nlocal : -1; }

int hvd_allreduce(hvd_comm* c, const hvd_tensor* t, int n, int op, uint64_t fusion_threshold, void* stream) {
  return traced(c, "ALLREDUCE", (uint64_t)n, list_bytes(t, n),
                [&] { return do_allreduce(c, t, n, op, fusion_threshold, static_cast<cudaStream_t>(stream)); });
}

// Host-buffer allreduce: chunk i is copied in (copy stream 1), reduced on the
// caller's stream by the same path as hvd_allreduce, and copied out (copy
// stream 2) while chunk i+1 is copied in — PCIe in, the ring, and PCIe out
// overlap through kHostSlots device staging slots.
// Every buffer is page-locked host memory the device reaches at the same address (UVA):
// the kernels can read / write it directly.
static bool host_mapped(hvd_comm* c, const void* const* in, void* const* out, uint64_t bytes) {
  for (int l = 0; l < c->nlocal; ++l) {
    for (const void* p : {static_cast<const void*>(in[l]), static_cast<const void*>(out[l])}) {
      cudaPointerAttributes a;
      if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
      if (a.type != cudaMemoryTypeHost || a.devicePointer != p) return false;
      (void)bytes;
    }
  }
  return true;
}

static int allreduce_host_impl(hvd_comm* c, const void* const* in, void* const* out, uint64_t count, int dtype, int op,
                       uint64_t chunk_bytes, void* stream) {
  int st = check_live(c);
  if (st != HVD_OK) return st;
  const int esz = elem_size(dtype);
  if (esz == 0) return HVD_ERR_UNSUPPORTED;
  if (!in || !out) return HVD_ERR_INVALID;
  for (int l = 0; l < c->nlocal; ++l)
    if (count && (!in[l] || !out[l])) return HVD_ERR_INVALID;
  if (count == 0) return HVD_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(c->device));
  if (c->host_zero_copy && c->fused && host_mapped(c, in, out, count * (uint64_t)esz)) {
    // zero copy: pinned host memory the device addresses directly (UVA) — the kernels gather
    // the gradients from it and scatter the results into it over PCIe, inside the ring
    // itself: no staging, no copy pipeline fill or drain
    std::vector<hvd_tensor> ti(c->nlocal), to(c->nlocal);
    bool same = true;
    for (int l = 0; l < c->nlocal; ++l) {
      ti[l] = {const_cast<void*>(in[l]), count, (hvd_dtype)dtype, 0};
      to[l] = {out[l], count, (hvd_dtype)dtype, 0};
      same = same && in[l] == out[l];
    }
    return do_allreduce(c, ti.data(), 1, op, c->cap, s, 0, nullptr, same ? nullptr : to.data());
  }
  uint64_t chunk = chunk_bytes ? chunk_bytes : (8ull << 20);
  chunk = std::max<uint64_t>(kChunkQuantum, chunk / kChunkQuantum * kChunkQuantum);
  chunk = std::min<uint64_t>(chunk, c->cap);
  if (c->stage_chunk < chunk) {  // (re)allocate the staging slots
    CK(cudaDeviceSynchronize());
    for (int l = 0; l < c->nlocal; ++l) {
      if (c->stage[l]) CK(cudaFree(c->stage[l]));
      c->stage[l] = nullptr;
      CK(cudaMalloc(reinterpret_cast<void**>(&c->stage[l]), chunk * hvd_comm::kHostSlots));
    }
    c->stage_chunk = chunk;
  }
  if (!c->s_h2d) {
    CK(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
    for (int k = 0; k < hvd_comm::kHostSlots; ++k) {
      CK(cudaEventCreateWithFlags(&c->ev_in[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_red[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_out[k], cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming));
  }
  // the copies start after everything already on the caller's stream (earlier calls'
  // staging use included: their copy-outs were joined into it)
  CK(cudaEventRecord(c->ev_start, s));
  CK(cudaStreamWaitEvent(c->s_h2d, c->ev_start, 0));
  CK(cudaStreamWaitEvent(c->s_d2h, c->ev_start, 0));
  const uint64_t ce = chunk / esz;  // elements per chunk (slots are c->stage_chunk bytes apart)
  const uint64_t nchunks = (count + ce - 1) / ce;
  std::vector<hvd_tensor> t(c->nlocal);
  for (uint64_t i = 0; i < nchunks; ++i) {
    const int k = (int)(i % hvd_comm::kHostSlots);
    const uint64_t off = i * ce;
    const uint64_t n = std::min<uint64_t>(ce, count - off);
    if (i >= (uint64_t)hvd_comm::kHostSlots) CK(cudaStreamWaitEvent(c->s_h2d, c->ev_out[k], 0));  // slot free
    for (int l = 0; l < c->nlocal; ++l)
      CK(cudaMemcpyAsync(c->stage[l] + (uint64_t)k * c->stage_chunk, static_cast<const char*>(in[l]) + off * esz,
                         n * esz, cudaMemcpyHostToDevice, c->s_h2d));
    CK(cudaEventRecord(c->ev_in[k], c->s_h2d));
    CK(cudaStreamWaitEvent(s, c->ev_in[k], 0));
    for (int l = 0; l < c->nlocal; ++l) {
      t[l].data = c->stage[l] + (uint64_t)k * c->stage_chunk;
      t[l].count = n;
      t[l].dtype = (hvd_dtype)dtype;
    }
    st = do_allreduce(c, t.data(), 1, op, c->cap, s);
    if (st != HVD_OK) return st;
    CK(cudaEventRecord(c->ev_red[k], s));
    CK(cudaStreamWaitEvent(c->s_d2h, c->ev_red[k], 0));
    for (int l = 0; l < c->nlocal; ++l)
      CK(cudaMemcpyAsync(static_cast<char*>(out[l]) + off * esz, c->stage[l] + (uint64_t)k * c->stage_chunk,
                         n * esz, cudaMemcpyDeviceToHost, c->s_d2h));
    CK(cudaEventRecord(c->ev_out[k], c->s_d2h));
  }
  CK(cudaEventRecord(c->ev_done, c->s_d2h));
  CK(cudaStreamWaitEvent(s, c->ev_done, 0));  // completion = the caller's stream
  return HVD_OK;
}

int hvd_allreduce_ex(hvd_comm* c, const hvd_tensor* t, int n, int op, uint64_t fusion_threshold, int wire_dtype,
                     void* stream) {
  return traced(c, "ALLREDUCE", (uint64_t)n, list_bytes(t, n), [&] {
    return do_allreduce(c, t, n, op, fusion_threshold, static_cast<cudaStream_t>(stream), wire_dtype);
  });
}

int hvd_allreduce_host(hvd_comm* c, const void* const* in, void* const* out, uint64_t count, int dtype, int op,
                       uint64_t chunk_bytes, void* stream) {
  return traced(c, "ALLREDUCE_HOST", 1, count * (uint64_t)elem_size(dtype),
                [&] { return allreduce_host_impl(c, in, out, count, dtype, op, chunk_bytes, stream); });
}

// ---- registered tensors -------------------------------------------------------------------
namespace {
// cuMemGetAddressRange through the runtime's driver entry point: no link-time
// dependency on libcuda (the library must load on CPU-only hosts).
typedef CUresult (*MemGetAddressRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
MemGetAddressRangeFn mem_get_address_range() {
  static MemGetAddressRangeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &p, 12000, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<MemGetAddressRangeFn>(p);
  }
  return fn;
}

struct RegEntry {
  cudaIpcMemHandle_t handle;
  uint64_t offset;  // tensor address - allocation base
  uint64_t count;
  int32_t dtype;
  int32_t pid;      // owner process: the same process maps `addr` directly (peer access)
  uint64_t addr;    // tensor address in the owner process
};
constexpr uint32_t kRegMagic = 0x48565247u;  // "HVRG"
}  // namespace

int hvd_register_blob(hvd_comm* c, const hvd_tensor* t, int n, void* blob, uint64_t* len) {
  if (!c || !len || n < 0 || (n > 0 && !t)) return HVD_ERR_INVALID;
  if (c->closed) return HVD_ERR_CLOSED;
  const uint64_t need = 8 + (uint64_t)n * sizeof(RegEntry);
  if (!blob) {
    *len = need;
    return HVD_OK;
  }
  if (*len < need) return HVD_ERR_INVALID;
  char* p = static_cast<char*>(blob);
  const uint32_t magic = kRegMagic;
  const int32_t nn = n;
  std::memcpy(p, &magic, 4);
  std::memcpy(p + 4, &nn, 4);
  CK(cudaSetDevice(c->device));
  for (int k = 0; k < n; ++k) {
    RegEntry e;
    std::memset(&e, 0, sizeof(e));
    e.count = t[k].count;
    e.dtype = t[k].dtype;
    if (!c->virt && c->size > 1 && t[k].count) {
      CUdeviceptr base = 0;
      size_t size = 0;
      MemGetAddressRangeFn range = mem_get_address_range();
      if (!range || range(&base, &size, reinterpret_cast<CUdeviceptr>(t[k].data)) != CUDA_SUCCESS)
        return HVD_ERR_CUDA;
      CK(cudaIpcGetMemHandle(&e.handle, reinterpret_cast<void*>(base)));
      e.offset = reinterpret_cast<uint64_t>(t[k].data) - (uint64_t)base;
      e.pid = (int32_t)getpid();
      e.addr = reinterpret_cast<uint64_t>(t[k].data);
    }
    std::memcpy(p + 8 + (size_t)k * sizeof(RegEntry), &e, sizeof(e));
  }
  *len = need;
  return HVD_OK;
}

int hvd_register(hvd_comm* c, const hvd_tensor* t, int n, const void* blobs, uint64_t len_each, int* reg_id) {
  int st = check_live(c);
  if (st != HVD_OK) return st;
  if (!reg_id || n < 0 || (n > 0 && !t)) return HVD_ERR_INVALID;
  for (int k = 0; k < n; ++k) {
    if (elem_size(t[k].dtype) == 0) return HVD_ERR_UNSUPPORTED;
    for (int l = 0; l < c->nlocal; ++l) {
      const hvd_tensor& x = t[(size_t)l * n + k];
      if (x.count != t[k].count || x.dtype != t[k].dtype || (x.count && !x.data)) return HVD_ERR_INVALID;
    }
  }
  Registration R;
  R.n = n;
  R.own.assign(t, t + (size_t)n * c->nlocal);
  R.succ.resize((size_t)n * c->nlocal);
  if (c->virt || c->size == 1) {
    for (int l = 0; l < c->nlocal; ++l)
      for (int k = 0; k < n; ++k)
        R.succ[(size_t)l * n + k] = static_cast<char*>(t[(size_t)((l + 1) % c->nlocal) * n + k].data);
  } else {
    if (!blobs || len_each < 8 + (uint64_t)n * sizeof(RegEntry)) return HVD_ERR_INVALID;
    const char* p = static_cast<const char*>(blobs) + (size_t)((c->rank + 1) % c->size) * len_each;
    uint32_t magic;
    int32_t nn;
    std::memcpy(&magic, p, 4);
    std::memcpy(&nn, p + 4, 4);
    if (magic != kRegMagic || nn != n) return HVD_ERR_INVALID;
    CK(cudaSetDevice(c->device));
    for (int k = 0; k < n; ++k) {
      RegEntry e;
      std::memcpy(&e, p + 8 + (size_t)k * sizeof(RegEntry), sizeof(e));
      if (e.count != t[k].count || e.dtype != t[k].dtype) return HVD_ERR_INVALID;
      if (!e.count) {
        R.succ[k] = nullptr;
        continue;
      }
      if (e.pid == (int32_t)getpid()) {  // the successor runs in this process (peer access)
        R.succ[k] = reinterpret_cast<char*>(e.addr);
        continue;
      }
      const std::string hk(reinterpret_cast<const char*>(&e.handle), sizeof(e.handle));
      auto it = c->ipc_maps.find(hk);
      char* base = nullptr;
      if (it != c->ipc_maps.end()) {
        base = it->second;
      } else {
        void* ptr = nullptr;
        CK(cudaIpcOpenMemHandle(&ptr, e.handle, cudaIpcMemLazyEnablePeerAccess));
        base = static_cast<char*>(ptr);
        c->ipc_maps[hk] = base;
      }
      R.succ[k] = base + e.offset;
    }
  }
  R.live = true;
  c->regs.push_back(std::move(R));
  *reg_id = (int)c->regs.size() - 1;
  return HVD_OK;
}

int hvd_allreduce_registered(hvd_comm* c, int reg_id, int op, uint64_t fusion_threshold, void* stream) {
  if (!c || reg_id < 0 || reg_id >= (int)c->regs.size() || !c->regs[reg_id].live) return HVD_ERR_INVALID;
  const Registration& R = c->regs[reg_id];
  return traced(c, "ALLREDUCE", (uint64_t)R.n, list_bytes(R.own.data(), R.n), [&] {
    return do_allreduce(c, R.own.data(), R.n, op, fusion_threshold, static_cast<cudaStream_t>(stream), 0,
                        c->size > 1 ? &R : nullptr);
  });
}

int hvd_allreduce_negotiated(hvd_comm* c, hvd_negotiator* g, const hvd_tensor* tensors, uint32_t n, int op,
                             uint64_t fusion_threshold, void* stream, uint32_t* ids_out, uint32_t* n_out) {
  return allreduce_negotiated_impl(c, g, tensors, n, op, fusion_threshold, stream, ids_out, n_out);
}

static int allreduce_negotiated_impl(hvd_comm* c, hvd_negotiator* g, const hvd_tensor* tensors, uint32_t n, int op,
                             uint64_t fusion_threshold, void* stream, uint32_t* ids_out, uint32_t* n_out) {
  int st = check_live(c);
  if (st != HVD_OK) return st;
  if (!g || !ids_out || !n_out || (n > 0 && !tensors)) return HVD_ERR_INVALID;
  if (hvd_neg::size_of(g) != c->size || hvd_neg::nlocal_of(g) != c->nlocal) return HVD_ERR_INVALID;
  std::vector<uint32_t> ids(hvd_neg::max_of(g));
  uint32_t m = 0;
  st = traced(c, "NEGOTIATE_ALLREDUCE", (uint64_t)n, 0, [&] {  // step 1: what is ready on every rank
    return hvd_negotiator_cycle(g, ids.data(), &m);
  });
  if (st != HVD_OK) {
    *n_out = m;
    return st;
  }
  if (c->jt && m > 0) {  // Horovod Timeline: each agreed tensor's negotiation phase
    std::vector<uint64_t> rec((size_t)3 * m);
    for (int l = 0; l < c->nlocal; ++l) {
      const uint32_t k = hvd_neg::trace_recent(g, l, m, rec.data());
      for (uint32_t i = 0; i < k; ++i)
        c->jt->negotiate(l, rec[3 * i], (int64_t)rec[3 * i + 1], (int64_t)rec[3 * i + 2]);
    }
  }
  std::vector<hvd_tensor> list((size_t)c->nlocal * m);
  for (uint32_t i = 0; i < m; ++i) {
    uint32_t id = 0;
    uint64_t count = 0;
    int dtype = 0;
    hvd_neg::agreed_meta(g, i, &id, &count, &dtype);
    if (id >= n) return HVD_ERR_INVALID;
    for (int l = 0; l < c->nlocal; ++l) {
      const hvd_tensor& t = tensors[(size_t)l * n + id];
      if (t.count != count || t.dtype != dtype) return HVD_ERR_INVALID;
      list[(size_t)l * m + i] = t;
    }
    ids_out[i] = id;
  }
  *n_out = m;
  if (m == 0) return HVD_OK;
  // steps 2-6 on the agreed tensors, in rank 0's submission order
  return traced(c, "ALLREDUCE", (uint64_t)m, list_bytes(list.data(), (int)m), [&] {
    return do_allreduce(c, list.data(), (int)m, op, fusion_threshold, static_cast<cudaStream_t>(stream));
  });
}

int hvd_deregister(hvd_comm* c, int reg_id) {
  if (!c || reg_id < 0 || reg_id >= (int)c->regs.size()) return HVD_ERR_INVALID;
  c->regs[reg_id].live = false;  // mapped peer allocations stay open until hvd_finalize
  return HVD_OK;
}

int hvd_allreduce_average(hvd_comm* c, const hvd_tensor* t, int n, uint64_t fusion_threshold, void* stream) {
  return traced(c, "ALLREDUCE", (uint64_t)n, list_bytes(t, n), [&] {
    return do_allreduce(c, t, n, HVD_AVERAGE, fusion_threshold, static_cast<cudaStream_t>(stream));
  });
}

int hvd_allreduce_buffer(hvd_comm* c, uint64_t count, int dtype, int op, void* stream) {
  return traced(c, "ALLREDUCE_BUFFER", 1, count * (uint64_t)elem_size(dtype),
                [&] { return allreduce_buffer_impl(c, count, dtype, op, stream); });
}

int hvd_broadcast(hvd_comm* c, const hvd_tensor* t, int n, int root, void* stream) {
  return traced(c, "BROADCAST", (uint64_t)n, list_bytes(t, n), [&] { return broadcast_impl(c, t, n, root, stream); });
}

int hvd_allgather(hvd_comm* c, const hvd_tensor* in, const hvd_tensor* out, void* stream) {
  return traced(c, "ALLGATHER", 1, list_bytes(in, 1), [&] { return allgather_impl(c, in, out, stream); });
}

static int allreduce_buffer_impl(hvd_comm* c, uint64_t count, int dtype, int op, void* stream) {
  int st = check_live(c);
  if (st != HVD_OK) return st;
  const int esz = elem_size(dtype);
  if (esz == 0) return HVD_ERR_UNSUPPORTED;
  if (op != HVD_SUM && op != HVD_AVERAGE) return HVD_ERR_INVALID;
  if (op == HVD_AVERAGE && (dtype == HVD_INT32 || dtype == HVD_INT64)) return HVD_ERR_UNSUPPORTED;
  if (count > c->cap / esz) return HVD_ERR_INVALID;
  if (count == 0) return HVD_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(c->device));
  if (c->fused) {
    // the fusion buffer itself is the single member, reduced in place by the fused
    // kernel as a registered tensor (the successor's buffer is already mapped), so the
    // kernel's channel-private use of the buffer region never touches it
    c->bufreg.n = 1;
    c->bufreg.own.resize(c->nlocal);
    c->bufreg.succ.resize(c->nlocal);
    for (int l = 0; l < c->nlocal; ++l) {
      c->bufreg.own[l] = {c->rk[l].buf, count, dtype, 0};
      c->bufreg.succ[l] = c->rk[l].nbuf;
    }
    c->bufreg.live = true;
    return do_allreduce(c, c->bufreg.own.data(), 1, op, c->cap, s, 0, c->size > 1 ? &c->bufreg : nullptr);
  }
  if (op == HVD_AVERAGE && c->size > 1) {  // N = 1: x * 1 = x (R1)
    char* bufs[kMaxLocal];
    for (int l = 0; l < c->nlocal; ++l) bufs[l] = c->rk[l].buf;
    JtRef jt;
    st = launch_counted(c, HVD_KERNEL_SCALE, s, &jt, count * esz, [&] {
      return launch_scale(bufs, c->nlocal, count, dtype, 1.0f / (float)c->size, pack_grid(c), kPackThreads, jt, s);
    });
    if (st != HVD_OK) return st;
  }
  return enqueue_ring(c, count, dtype, s);
}

void* hvd_fusion_buffer(hvd_comm* c, int local) {
  if (!c || c->closed || local < 0 || local >= c->nlocal) return nullptr;
  return c->rk[local].buf;
}

uint64_t hvd_fusion_capacity(const hvd_comm* c) { return c ? c->cap : 0; }

static int broadcast_impl(hvd_comm* c, const hvd_tensor* t, int n, int root, void* stream) {
  int st = check_live(c);
  if (st != HVD_OK) return st;
  if (root < 0 || root >= c->size || n < 0 || (n > 0 && !t)) return HVD_ERR_INVALID;
  for (int k = 0; k < n; ++k) {
    if (elem_size(t[k].dtype) == 0) return HVD_ERR_UNSUPPORTED;
    for (int l = 0; l < c->nlocal; ++l) {
      const hvd_tensor& x = t[(size_t)l * n + k];
      if (x.count != t[k].count || x.dtype != t[k].dtype) return HVD_ERR_INVALID;
      if (x.count && !x.data) return HVD_ERR_INVALID;
    }
  }
  if (n == 0 || c->size == 1) return HVD_OK;  // N = 1: the root's tensors are the result
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(c->device));
  CachedPlan* plan = nullptr;
  st = get_plan(c, t, n, c->cap, s, &plan);  // fuse the tensors into as few buffers as possible
  if (st != HVD_OK) return st;
  for (DevPlanBuffer& b : plan->bufs) {
    if (b.L == 0) continue;
    const uint64_t g = kChunkQuantum / elem_size(b.dtype);
    FusedParams F;
    std::memset(&F, 0, sizeof(F));
    int nch = 0;
    st = make_ring_params(c, b.L, b.dtype, true, &F.ring, &nch, (b.L + g - 1) / g * g);  // one chunk
    if (st != HVD_OK) return st;
    F.ring.mode = kRingBroadcast;
    F.ring.root = root;
    F.ring.epoch = ++c->hs_epoch;
    F.segs = b.pp.segs;
    F.src = b.pp.src;
    F.dst = nullptr;
    F.vbeg_global = b.vbeg;
    F.nseg = b.pp.nseg;
    F.dtype = b.dtype;
    st = launch_counted(c, HVD_KERNEL_COPY, s, &F.ring.jt, fused_bytes(F), [&] { return launch_copy(F, b.dtype, nch, c->nlocal, c->threads, s); });
    if (st != HVD_OK) return st;
    const unsigned long long inc = ring_signals(kRingBroadcast, c->size, F.ring.K);
    for (int ch = 0; ch < nch; ++ch) c->base[ch] += inc;
  }
  return HVD_OK;
}

static int allgather_impl(hvd_comm* c, const hvd_tensor* in, const hvd_tensor* out, void* stream) {
  int st = check_live(c);
  if (st != HVD_OK) return st;
  if (!in || !out) return HVD_ERR_INVALID;
  const int dtype = in[0].dtype;
  const int esz = elem_size(dtype);
  if (esz == 0) return HVD_ERR_UNSUPPORTED;
  const uint64_t count = in[0].count;
  const int N = c->size;
  for (int l = 0; l < c->nlocal; ++l) {
    if (in[l].count != count || in[l].dtype != dtype || out[l].dtype != dtype) return HVD_ERR_INVALID;
    if (out[l].count != count * (uint64_t)N) return HVD_ERR_INVALID;
    if (count && (!in[l].data || !out[l].data)) return HVD_ERR_INVALID;
  }
  if (count == 0) return HVD_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(c->device));
  const uint64_t g = kChunkQuantum / esz;
  const uint64_t m_max = c->cap / ((uint64_t)N * esz) / g * g;  // elements per rank per piece
  if (m_max == 0) return HVD_ERR_INVALID;
  const uint64_t vel = kPackVecBytes / esz;
  for (uint64_t off = 0; off < count; off += m_max) {
    const uint64_t m = std::min(m_max, count - off);
    const uint64_t qpad = (m + g - 1) / g * g;  // block b of the buffer at b * qpad
    std::vector<uint64_t> key = {0x41475448ull /* "AGTH" */, (uint64_t)c->nlocal, count, (uint64_t)dtype, off, m};
    for (int l = 0; l < c->nlocal; ++l) {
      key.push_back(reinterpret_cast<uint64_t>(in[l].data));
      key.push_back(reinterpret_cast<uint64_t>(out[l].data));
    }
    CachedPlan* plan = lookup_plan(c, key);
    if (!plan) {
      std::vector<HostBuf> hb(1);
      HostBuf& B = hb[0];
      B.dtype = dtype;
      B.L = (uint64_t)N * qpad;
      B.segs.resize(N);
      B.src.resize((size_t)N * c->nlocal);
      B.dst.resize((size_t)N * c->nlocal);
      for (int b = 0; b < N; ++b) {
        B.segs[b] = {(unsigned long long)b * qpad, m, (unsigned long long)b * qpad / vel, 0};
        for (int l = 0; l < c->nlocal; ++l) {
          B.src[(size_t)l * N + b] = static_cast<char*>(in[l].data) + off * esz;  // gathered for b == rank only
          B.dst[(size_t)l * N + b] = static_cast<char*>(out[l].data) + ((uint64_t)b * count + off) * esz;
        }
      }
      st = upload_plan(c, std::move(key), hb, s, &plan);
      if (st != HVD_OK) return st;
    }
    DevPlanBuffer& b = plan->bufs[0];
    FusedParams F;
    std::memset(&F, 0, sizeof(F));
    int nch = 0;
    st = make_ring_params(c, b.L, dtype, true, &F.ring, &nch, qpad);
    if (st != HVD_OK) return st;
    F.segs = b.pp.segs;
    F.src = b.pp.src;
    F.dst = b.dst;
    F.vbeg_global = b.vbeg;
    F.nseg = b.pp.nseg;
    F.dtype = dtype;
    if (N == 1) {  // out = in: the fused kernel's N = 1 path (gather -> scatter), no scale
      b.pp.scale_on = 0;
      b.pp.scale = 1.0f;
      DevPlanBuffer* one = &b;
      st = enqueue_fused_multi(c, &one, 1, s);
      if (st != HVD_OK) return st;
      continue;
    }
    F.ring.mode = kRingAllgather;
    F.ring.epoch = ++c->hs_epoch;
    st = launch_counted(c, HVD_KERNEL_COPY, s, &F.ring.jt, fused_bytes(F), [&] { return launch_copy(F, dtype, nch, c->nlocal, c->threads, s); });
    if (st != HVD_OK) return st;
    const unsigned long long inc = ring_signals(kRingAllgather, N, F.ring.K);
    for (int ch = 0; ch < nch; ++ch) c->base[ch] += inc;
  }
  return HVD_OK;
}

int hvd_poll_error(hvd_comm* c) {
  if (!c) return HVD_ERR_INVALID;
  if (c->closed) return HVD_ERR_CLOSED;
  return *c->err_host;
}

#ifndef HVD_BUILD_ID
#define HVD_BUILD_ID "hvd-src-unknown"
#endif
const char* hvd_build_id(void) { return HVD_BUILD_ID; }

const char* hvd_strerror(int status) {
  switch (status) {
    case HVD_OK: return "ok";
    case HVD_ERR_INVALID: return "invalid argument";
    case HVD_ERR_UNSUPPORTED: return "unsupported dtype/op combination";
    case HVD_ERR_CUDA: return "CUDA runtime error";
    case HVD_ERR_NOT_CONNECTED: return "communicator not connected";
    case HVD_ERR_TIMEOUT: return "device watchdog timeout (a peer did not signal)";
    case HVD_ERR_CLOSED: return "communicator finalized";
    case HVD_ERR_MISMATCH: return "ranks made different collective calls";
    default: return "unknown status";
  }
}

int hvd_traffic(hvd_comm* c, int local, uint64_t* sent_bytes, uint64_t* sends) {
  if (!c || local < 0 || local >= c->nlocal || !sent_bytes || !sends) return HVD_ERR_INVALID;
  if (c->closed) return HVD_ERR_CLOSED;
  unsigned long long v[2];
  CK(cudaSetDevice(c->device));
  CK(cudaMemcpy(v, c->rk[local].stats, sizeof(v), cudaMemcpyDeviceToHost));
  *sent_bytes = v[0];
  *sends = v[1];
  return HVD_OK;
}

int hvd_set_config(hvd_comm* c, int key, int64_t value) {
  if (!c) return HVD_ERR_INVALID;
  switch (key) {
    case HVD_CFG_CHANNELS:
      if (value < 1 || value > kMaxChannels) return HVD_ERR_INVALID;
      c->channels = (int)value;
      return HVD_OK;
    case HVD_CFG_SLICE_BYTES:
      if (value != 0 && (value < kChunkQuantum || value % kChunkQuantum)) return HVD_ERR_INVALID;
      c->slice_bytes = value;
      return HVD_OK;
    case HVD_CFG_THREADS:
      if (value < 64 || value > 384 || value % 32 || value + 32 * c->sig_warps > kMaxRingThreads + 32)
        return HVD_ERR_INVALID;
      c->threads = (int)value;
      return HVD_OK;
    case HVD_CFG_TIMEOUT_MS:
      if (value < 1) return HVD_ERR_INVALID;
      c->timeout_ms = value;
      return HVD_OK;
    case HVD_CFG_PACK_CTAS_PER_SM:
      if (value < 1 || value > 8) return HVD_ERR_INVALID;
      c->pack_ctas_per_sm = (int)value;
      return HVD_OK;
    case HVD_CFG_PROFILE:
      if (value != 0 && value != 1) return HVD_ERR_INVALID;
      c->profile = (int)value;
      return HVD_OK;
    case HVD_CFG_SIGNAL_MODE:
      if (value < 1 || value > 2) return HVD_ERR_INVALID;
      c->sig_mode = (int)value;
      return HVD_OK;
    case HVD_CFG_FUSED:
      if (value != 0 && value != 1) return HVD_ERR_INVALID;
      c->fused = (int)value;
      return HVD_OK;
    case HVD_CFG_LL_MAX_BYTES:
      if (value < 0 || value > (int64_t)kLLLimitBytes) return HVD_ERR_INVALID;
      c->ll_max = value;
      return HVD_OK;
    case HVD_CFG_LL128_MAX_BYTES:
      if (value < 0 || value > (int64_t)kLL128LimitBytes) return HVD_ERR_INVALID;
      c->ll128_max = value;
      return HVD_OK;
    case HVD_CFG_MULTI_BUFFERS:
      if (value < 1 || value > kMaxMultiBufs) return HVD_ERR_INVALID;
      c->multi_bufs = (int)value;
      return HVD_OK;
    case HVD_CFG_PROTOCOL:
      if (value < 0 || value > 2) return HVD_ERR_INVALID;
      if (value == 0 && c->size > 1 && !c->pull_ok) {
        // the pull protocol reads the predecessor's pull buffers: virtual mode allocates
        // them now; a real rank needs HVD_CFG_PULL_BUFFERS on every rank before connecting
        if (!c->virt) return HVD_ERR_INVALID;
        const int st = alloc_pull(c);
        if (st != HVD_OK) return st;
      }
      c->protocol = (int)value;
      return HVD_OK;
    case HVD_CFG_PULL_BUFFERS:
      if (value != 0 && value != 1) return HVD_ERR_INVALID;
      if (value == 0) return (c->pull_mem[0] || (c->want_pull && c->blob_out)) ? HVD_ERR_INVALID : (c->want_pull = false, HVD_OK);
      if (c->virt) return alloc_pull(c);
      if (c->blob_out) return c->want_pull ? HVD_OK : HVD_ERR_INVALID;
      c->want_pull = true;
      return HVD_OK;
    case HVD_CFG_SOLO_KERNEL:
      if (value != 0 && value != 1) return HVD_ERR_INVALID;
      c->solo_kernel = (int)value;
      return HVD_OK;
    case HVD_CFG_SOLO_STAGES:
      if (value < 2 || value > 8 || bulk_smem_bytes((int)value, c->solo_stage_bytes, false) > kBulkMaxSmem)
        return HVD_ERR_INVALID;
      c->solo_stages = (int)value;
      return HVD_OK;
    case HVD_CFG_LL_PDL:
      if (value < 0 || value > 1) return HVD_ERR_INVALID;
      c->ll_pdl = (int)value;
      return HVD_OK;
    case HVD_CFG_PREISSUE:
      if (value < -1 || value > 1) return HVD_ERR_INVALID;
      c->preissue = (int)value;
      return HVD_OK;
    case HVD_CFG_HOST_ZERO_COPY:
      if (value < 0 || value > 1) return HVD_ERR_INVALID;
      c->host_zero_copy = (int)value;
      return HVD_OK;
    case HVD_CFG_WATCHER:
      if (value < 0 || value > 1) return HVD_ERR_INVALID;
      c->watcher = (int)value;
      return HVD_OK;
    case HVD_CFG_FUSED_PDL:
      if (value < 0 || value > 2) return HVD_ERR_INVALID;
      c->fused_pdl = (int)value;
      return HVD_OK;
    case HVD_CFG_PACE_GBPS:
      if (value < 0 || value > 100000) return HVD_ERR_INVALID;
      c->pace_gbps = (int)value;
      return HVD_OK;
    case HVD_CFG_PACE_BURST_ROWS:
      if (value < 0 || value > 1024) return HVD_ERR_INVALID;
      c->pace_burst_rows = (int)value;
      return HVD_OK;
    case HVD_CFG_SOLO_TAIL:
      if (value < -1) return HVD_ERR_INVALID;
      c->solo_tail = value;
      CK(cudaSetDevice(c->device));
      drop_plans(c->cache);  // member tables are built with the plan
      return HVD_OK;
    case HVD_CFG_SOLO_STAGE_BYTES:
      if (value < (4 << 10) || value > (64 << 10) || value % 1024 ||
          bulk_smem_bytes(c->solo_stages, (int)value, false) > kBulkMaxSmem)
        return HVD_ERR_INVALID;
      c->solo_stage_bytes = (int)value;
      return HVD_OK;
    case HVD_CFG_SIGNAL_WARPS:
      if (value < 1 || value > 4 || c->threads + 32 * value > kMaxRingThreads + 32) return HVD_ERR_INVALID;
      c->sig_warps = (int)value;
      return HVD_OK;
    case HVD_CFG_BULK_STAGES:
      if (value < 2 || value > 8 ||
          bulk_smem_bytes((int)value, c->bulk_stage_bytes) > kBulkMaxSmem)
        return HVD_ERR_INVALID;
      c->bulk_stages = (int)value;
      return HVD_OK;
    case HVD_CFG_BULK_STAGE_BYTES:
      if (value < (4 << 10) || value > (64 << 10) || value % 1024 ||
          bulk_smem_bytes(c->bulk_stages, (int)value) > kBulkMaxSmem)
        return HVD_ERR_INVALID;
      c->bulk_stage_bytes = (int)value;
      return HVD_OK;
    case HVD_CFG_BULK_DEPTH:
      if (value < 0 || value > 3) return HVD_ERR_INVALID;
      c->bulk_depth = (int)value;
      return HVD_OK;
    case HVD_CFG_BULK_CHANNELS:
      if (value < 1 || value > kMaxChannels) return HVD_ERR_INVALID;
      c->bulk_channels = (int)value;
      return HVD_OK;
    case HVD_CFG_BULK_SLICE_BYTES:
      if (value < kChunkQuantum || value % kChunkQuantum) return HVD_ERR_INVALID;
      c->bulk_slice = value;
      return HVD_OK;
    case HVD_CFG_WINDOW:
      if (value < 0 || value > 1024) return HVD_ERR_INVALID;
      c->window = (int)value;
      return HVD_OK;
    case HVD_CFG_FIN_LAG:
      if (value < 0 || value > 1 << 20) return HVD_ERR_INVALID;
      c->fin_lag = (int)value;
      return HVD_OK;
    case HVD_CFG_TIMELINE: {
      if (value < 0 || value > 65536) return HVD_ERR_INVALID;
      CK(cudaSetDevice(c->device));
      CK(cudaDeviceSynchronize());
      if (c->tl) cudaFree(c->tl);
      c->tl = nullptr;
      c->tl_max = (int)value;
      c->tl_slices = 0;
      if (value > 0) {
        const size_t bytes = tl_words(c->tl_max) * c->nlocal * sizeof(unsigned long long);
        CK(cudaMalloc(reinterpret_cast<void**>(&c->tl), bytes));
        CK(cudaMemset(c->tl, 0, bytes));
      }
      return HVD_OK;
    }
    default: return HVD_ERR_INVALID;
  }
}

int64_t hvd_get_config(const hvd_comm* c, int key) {
  if (!c) return -1;
  switch (key) {
    case HVD_CFG_CHANNELS: return c->channels;
    case HVD_CFG_SLICE_BYTES: return c->slice_bytes;
    case HVD_CFG_THREADS: return c->threads;
    case HVD_CFG_TIMEOUT_MS: return c->timeout_ms;
    case HVD_CFG_PACK_CTAS_PER_SM: return c->pack_ctas_per_sm;
    case HVD_CFG_PROFILE: return c->profile;
    case HVD_CFG_SIGNAL_MODE: return c->sig_mode;
    case HVD_CFG_FUSED: return c->fused;
    case HVD_CFG_TIMELINE: return c->tl_max;
    case HVD_CFG_WINDOW: return c->window;
    case HVD_CFG_PROTOCOL: return c->protocol;
    case HVD_CFG_PULL_BUFFERS: return (c->pull_ok || c->want_pull) ? 1 : 0;
    case HVD_CFG_MULTI_BUFFERS: return c->multi_bufs;
    case HVD_CFG_LL_MAX_BYTES: return c->ll_max;
    case HVD_CFG_LL128_MAX_BYTES: return c->ll128_max;
    case HVD_CFG_FIN_LAG: return c->fin_lag;
    case HVD_CFG_SIGNAL_WARPS: return c->sig_warps;
    case HVD_CFG_LL128_STATUS: return c->ll128_status;
    case HVD_CFG_SOLO_KERNEL: return c->solo_kernel;
    case HVD_CFG_SOLO_STAGES: return c->solo_stages;
    case HVD_CFG_PACE_GBPS: return c->pace_gbps;
    case HVD_CFG_FUSED_PDL: return c->fused_pdl;
    case HVD_CFG_WATCHER: return c->watcher;
    case HVD_CFG_HOST_ZERO_COPY: return c->host_zero_copy;
    case HVD_CFG_PREISSUE: return c->preissue;
    case HVD_CFG_LL_PDL: return c->ll_pdl;
    case HVD_CFG_PACE_BURST_ROWS: return c->pace_burst_rows;
    case HVD_CFG_SOLO_STAGE_BYTES: return c->solo_stage_bytes;
    case HVD_CFG_SOLO_TAIL: return c->solo_tail;
    case HVD_CFG_BULK_STAGES: return c->bulk_stages;
    case HVD_CFG_BULK_STAGE_BYTES: return c->bulk_stage_bytes;
    case HVD_CFG_BULK_DEPTH: return c->bulk_depth;
    case HVD_CFG_BULK_CHANNELS: return c->bulk_channels;
    case HVD_CFG_BULK_SLICE_BYTES: return c->bulk_slice;
    default: return -1;
  }
}

int hvd_timeline(hvd_comm* c, int local, uint64_t* out, uint64_t cap_words, hvd_timeline_info* info) {
  if (!c || !info || local < 0 || local >= c->nlocal) return HVD_ERR_INVALID;
  if (c->closed) return HVD_ERR_CLOSED;
  std::memset(info, 0, sizeof(*info));
  if (!c->tl || c->tl_slices == 0) return HVD_OK;
  info->channels = c->tl_nch;
  info->slices = std::min(c->tl_slices, c->tl_max);
  info->signals = std::min(c->tl_T * c->tl_K, c->tl_max);
  info->kind = c->tl_kind;  // 0: push/fused kernel records, 1: pull kernel records
  info->K = c->tl_K;
  info->T = c->tl_T;
  info->rank = c->virt ? local : c->rank;
  info->size = c->size;
  info->words_per_channel = (uint64_t)c->tl_max * 2;
  const size_t words = tl_words(c->tl_max);
  if (!out) return HVD_OK;
  if (cap_words < words) return HVD_ERR_INVALID;
  CK(cudaSetDevice(c->device));
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(out, c->tl + words * local, words * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return HVD_OK;
}

int hvd_timeline_start(hvd_comm* c, const char* path, int truncate) {
  int st = check_live(c);
  if (st != HVD_OK) return st;
  if (!path || !path[0] || c->jt) return HVD_ERR_INVALID;
  return timeline_start(c, path, truncate != 0);
}

int hvd_timeline_stop(hvd_comm* c) {
  if (!c) return HVD_ERR_INVALID;
  if (c->closed) return HVD_ERR_CLOSED;
  if (!c->jt) return HVD_OK;
  CK(cudaSetDevice(c->device));
  const int st = cuda_fail(cudaDeviceSynchronize(), "timeline stop");
  c->jt->drain(true);
  delete c->jt;
  c->jt = nullptr;
  return st;
}

int hvd_timeline_flush(hvd_comm* c, uint64_t* launches, uint64_t* dropped) {
  if (!c) return HVD_ERR_INVALID;
  if (c->closed) return HVD_ERR_CLOSED;
  if (launches) *launches = c->jt ? c->jt->launches() : 0;
  if (dropped) *dropped = c->jt ? c->jt->dropped() : 0;
  if (!c->jt) return HVD_OK;
  c->jt->drain(false);
  c->jt->flush();
  return HVD_OK;
}

int hvd_kernel_stats(hvd_comm* c, uint64_t* launches, double* device_ms) {
  if (!c || !launches || !device_ms) return HVD_ERR_INVALID;
  if (c->closed) return HVD_ERR_CLOSED;
  for (int k = 0; k < HVD_KERNEL_KINDS; ++k) {
    launches[k] = c->launches[k];
    device_ms[k] = 0.0;
    c->launches[k] = 0;
  }
  int st = HVD_OK;
  for (auto& t : c->timed) {
    float ms = 0.f;
    if (st == HVD_OK && cudaEventSynchronize(t.b) == cudaSuccess &&
        cudaEventElapsedTime(&ms, t.a, t.b) == cudaSuccess)
      device_ms[t.kind] += ms;
    else
      st = HVD_ERR_CUDA;
    c->event_pool.push_back(t.a);
    c->event_pool.push_back(t.b);
  }
  c->timed.clear();
  return st;
}

}  // extern "C"

/*
 * hvd.h — C ABI of the B200-native fused ring allreduce (Horovod, arXiv 1802.05799).
 *
 * The library implements the data-parallel hot path of the paper:
 *   Tensor Fusion (§7): pack many gradient tensors into a
 *   fusion buffer, fused with the averaging scale 1/N, run the ring
 *   allreduce on the buffer, unpack the result into the tensors;
 *   ring-allreduce (§3): N-1 reduce-scatter iterations in
 *   which "received values are added", then N-1 all-gather iterations in which
 *   "received values replace", each rank talking only to its ring neighbours.
 * The API follows the paper's four user calls:
 * init, allreduce-average of the gradients, broadcast of the initial state,
 * plus allgather (north_star).
 *
 * Conventions
 *   - Every call returns an hvd_status (0 = OK, < 0 = error); nothing throws or
 *     aborts across the ABI.  Argument errors are reported synchronously and
 *     leave the communicator unchanged.  Device-side errors (the spin-wait
 *     watchdog) are asynchronous: they are latched in host-mapped memory and
 *     returned by hvd_poll_error() and by every later call on that comm.
 *   - Device pointers are plain CUDA device addresses on the comm's device.
 *     Streams are cudaStream_t passed as void* (NULL = legacy default stream).
 *     Work is enqueued on the stream and the call returns without a host
 *     synchronisation (stream-ordered completion, north_star); the caller's
 *     tensors must stay valid and unmodified until that work completes.
 *   - Ownership: the caller owns its tensors; the library owns the fusion
 *     buffer, the reduce-scatter scratch, the signal flags and the peer
 *     mappings ("Allocate a fusion buffer if it was not previously
 *     allocated"), all released by hvd_finalize.
 *   - Collective contract: every rank makes the same sequence of collective
 *     calls with identical tensor counts, dtypes, op, threshold and root.  A
 *     ring launch whose geometry differs between neighbours is caught by the
 *     launch handshake (HVD_ERR_MISMATCH, async); other mismatches wait until
 *     the watchdog fires (HVD_ERR_TIMEOUT).  Neither corrupts memory silently
 *     nor hangs the GPU.
 *   - A comm is not thread-safe; use one comm per thread.
 *
 * Virtual ranks: hvd_init_virtual() creates a comm that simulates all N ranks
 * on ONE device (one kernel launch spans every rank, so the ranks' CTAs are
 * co-resident).  It runs exactly the same kernels and signal protocol as the
 * multi-process path, with "peer" pointers that are same-device buffers.  In
 * that mode every tensor-list argument holds the lists of all local ranks,
 * rank-major: element [r * n + k] is tensor k of rank r.
 */
#ifndef HVD_B200_H
#define HVD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HVD_ABI_VERSION 3

typedef enum {
  HVD_OK = 0,
  HVD_ERR_INVALID = -1,        /* bad argument (null pointer, size, rank, count overflow) */
  HVD_ERR_UNSUPPORTED = -2,    /* e.g. AVERAGE on an integer dtype      */
  HVD_ERR_CUDA = -3,           /* a CUDA runtime call failed                              */
  HVD_ERR_NOT_CONNECTED = -4,  /* size > 1 and hvd_connect() has not completed            */
  HVD_ERR_TIMEOUT = -5,        /* a device spin-wait exceeded the watchdog (async)        */
  HVD_ERR_CLOSED = -6,         /* comm already finalized                                  */
  HVD_ERR_MISMATCH = -7        /* ranks made different collective calls (async): the launch
                                  handshake carries a hash of the call's geometry and the
                                  successor's must equal this rank's                       */
} hvd_status;

typedef enum { HVD_FLOAT32 = 1, HVD_BFLOAT16 = 2, HVD_INT32 = 3, HVD_INT64 = 4 } hvd_dtype;
typedef enum { HVD_SUM = 0, HVD_AVERAGE = 1 } hvd_op;

/* A flat, contiguous tensor in device memory.  count == 0 is a legal no-op. */
typedef struct {
  void* data;      /* device pointer (any alignment; 16 B alignment is the fast path) */
  uint64_t count;  /* elements */
  int32_t dtype;   /* hvd_dtype */
  int32_t reserved;
} hvd_tensor;

typedef struct hvd_comm hvd_comm; /* opaque */

/* ---- lifecycle ("hvd.init() initializes Horovod") ------------------------ */

/* Create the comm of ring rank `rank` of `size` on CUDA device `device` and
 * allocate its fusion buffer of `fusion_bytes` (0 = default 64 MiB, P:L368-369;
 * rounded up to 4 KiB).  One device region holds it together with two
 * reduce-scatter scratch halves, the signal / ready / hash words and the LL
 * region.  Each region buffer is sized 3x the capacity (capacity <= 256 MiB) so
 * that the buffers of a multi-buffer call fit side by side, plus a 416 MiB LL /
 * LL128 region: 998 MiB at the default.  The pull protocol's two buffers (2 x
 * 194 MiB) are allocated only when it is enabled (HVD_CFG_PULL_BUFFERS; the
 * environment variable HVD_PULL_BUFFERS=1 sets it at init).  For size > 1 the
 * comm must then exchange blobs and hvd_connect().
 * Errors: INVALID (size < 1, rank out of range, null out), CUDA. */
int hvd_init(int rank, int size, int device, uint64_t fusion_bytes, hvd_comm** out);

/* Create a comm that simulates all `size` ranks on one device (see header
 * comment).  It is connected on return.  Errors: INVALID (size < 1 or > 8), CUDA. */
int hvd_init_virtual(int size, int device, uint64_t fusion_bytes, hvd_comm** out);

/* Bootstrap: write this rank's CUDA-IPC blob into `out` (caller-owned,
 * *len bytes).  With out == NULL only *len (the blob size) is returned.  The
 * caller gathers the blobs of all ranks in rank order (any transport) and
 * passes them to hvd_connect.  Errors: INVALID (len too small). */
int hvd_get_ipc_blob(hvd_comm* c, void* out, uint64_t* len);

/* Map the ring successor's buffers from the gathered blobs
 * (`blobs` = size * len_each bytes, rank order).  Must be called on every
 * rank; the caller must barrier all ranks after it before the first
 * collective.  A peer in another process is mapped by CUDA IPC; a peer in the
 * SAME process (one process driving several GPUs, each with its own comm) by
 * peer access to its allocation — then the ranks' hvd_connect calls must run
 * concurrently (one thread each: the call ends with a collective self-test).
 * Errors: INVALID (blob mismatch), CUDA (IPC open / peer access failed). */
int hvd_connect(hvd_comm* c, const void* blobs, uint64_t len_each);

/* Release everything.  Idempotent on a NULL comm; waits for the device.  */
int hvd_finalize(hvd_comm* c);

int hvd_rank(const hvd_comm* c);        /* ring rank (virtual comm: 0)                */
int hvd_size(const hvd_comm* c);        /* N                                          */
int hvd_local_ranks(const hvd_comm* c); /* ranks driven by this comm (1 or N)         */

/* ---- the hot path ---------------------------------------------------------------------------- */

/* In-place allreduce of the n tensors `t` (n per local rank, see header).
 * Tensor Fusion: tensors are grouped next-fit in the given order
 * into fusion buffers of at most min(fusion_threshold, capacity) bytes (16 B
 * aligned members, same dtype; fusion_threshold == 0 turns fusion off; a tensor
 * larger than the limit is split into limit-sized segments — DESIGN.md R6-R8).
 * Per buffer: pack (with x * fl32(1/N) for AVERAGE, R1) -> ring reduce-scatter
 * + all-gather -> unpack, all enqueued on `stream`.  How (same
 * bits every way): by default one persistent launch per call gathers in the
 * first ring step and scatters in the all-gather steps (zero-copy, all buffers
 * of the call pipelined); buffers up to HVD_CFG_LL_MAX_BYTES (or 256 KiB / 1 MiB at N = 2 / N > 2 in a
 * multi-buffer call) take the LL latency protocol — except that in a call of at most 16
 * buffers with a buffer for the persistent launch, small buffers of the same dtype join
 * that launch — and a lone buffer up to HVD_CFG_LL128_MAX_BYTES the LL128 protocol; at
 * N = 1 a plain HBM stream.
 * op: HVD_SUM (all dtypes) or HVD_AVERAGE (float dtypes only).
 * Errors: INVALID (null/size), UNSUPPORTED (AVERAGE on integers, bad dtype),
 * NOT_CONNECTED, TIMEOUT / MISMATCH (latched), CUDA. */
int hvd_allreduce(hvd_comm* c, const hvd_tensor* t, int n, int op, uint64_t fusion_threshold,
                  void* stream);

/* hvd_allreduce with a wire dtype (R14): the fusion buffer
 * and every ring step use `wire_dtype` instead of the tensors' dtype.  All n
 * tensors must share one float dtype; wire_dtype is HVD_FLOAT32 or HVD_BFLOAT16
 * (0 or the tensors' dtype = plain hvd_allreduce).  fp32 tensors over a bf16
 * wire: pack rounds fl32(x*s) to bf16 RNE (half the NVLink bytes), unpack
 * widens exactly; bf16 tensors over an fp32 wire: fp32 partials, one final
 * RNE rounding.  Fusion limits count wire bytes.  Needs HVD_CFG_FUSED=1.
 * Errors: as hvd_allreduce; UNSUPPORTED for mixed or integer tensor dtypes. */
int hvd_allreduce_ex(hvd_comm* c, const hvd_tensor* t, int n, int op, uint64_t fusion_threshold,
                     int wire_dtype, void* stream);

/* ---- registered tensors: zero-copy both ways (SURVEY §8f-1 "the last AG step writes
 * straight into outputs") ----------------------------------------------------------------
 * A training loop reduces the same gradient tensors every step.  Registering them
 * once maps every rank's tensors into its predecessor (CUDA IPC), so the all-gather
 * iterations write the final values directly into the successor's tensors: no
 * fusion-buffer forward and no final unpack.  Same ring order, same bits.
 * Collective: every rank registers the same list shape.  Bootstrap like hvd_init:
 * hvd_register_blob (blob == NULL -> *len only) -> gather the blobs of all ranks
 * (rank order) -> hvd_register (virtual comms: blobs may be NULL).  The tensors
 * must stay allocated until hvd_deregister / hvd_finalize.
 * Errors: INVALID (shape mismatch across ranks, bad id), CUDA (IPC).             */
int hvd_register_blob(hvd_comm* c, const hvd_tensor* t, int n, void* blob, uint64_t* len);
int hvd_register(hvd_comm* c, const hvd_tensor* t, int n, const void* blobs, uint64_t len_each,
                 int* reg_id);
/* In-place allreduce of registered tensor list `reg_id` (op, fusion as hvd_allreduce). */
int hvd_allreduce_registered(hvd_comm* c, int reg_id, int op, uint64_t fusion_threshold,
                             void* stream);
int hvd_deregister(hvd_comm* c, int reg_id);

/* hvd_allreduce(c, t, n, HVD_AVERAGE, fusion_threshold, stream): the paper's
 * "average gradients among those multiple copies". */
int hvd_allreduce_average(hvd_comm* c, const hvd_tensor* t, int n, uint64_t fusion_threshold,
                          void* stream);

/* Raw ring on the first `count` elements of the registered fusion buffer(s),
 * no pack/unpack (the headline 64 MiB measurement).  AVERAGE prescales in
 * place first.  count * esz must be <= capacity.  Same errors as above. */
int hvd_allreduce_buffer(hvd_comm* c, uint64_t count, int dtype, int op, void* stream);

/* Device address of local rank `local`'s fusion buffer (capacity bytes), NULL on error. */
void* hvd_fusion_buffer(hvd_comm* c, int local);
uint64_t hvd_fusion_capacity(const hvd_comm* c);

/* ---- broadcast and allgather (north_star) ---------------------------------------- */

/* Every rank's n tensors become bitwise copies of rank `root`'s (pipelined ring
 * forward through the fusion buffer).  Errors: INVALID (root), as above. */
int hvd_broadcast(hvd_comm* c, const hvd_tensor* t, int n, int root, void* stream);

/* out (size * in.count elements, same dtype) = concatenation of every rank's
 * `in` in rank order (ring all-gather, R12).  `in` and `out` hold one
 * tensor per local rank.  Errors: INVALID (out too small, dtype mismatch). */
int hvd_allgather(hvd_comm* c, const hvd_tensor* in, const hvd_tensor* out, void* stream);

/* ---- errors, statistics, tuning -------------------------------------------------------------- */

/* LL128 safety (HVD_CFG_LL128_MAX_BYTES): the LL128 protocol relies on a warp's 128-byte
 * line store arriving whole at the peer, which PTX does not promise.  hvd_connect runs
 * this check on every communicator of N > 1 processes; virtual comms may call it.
 * Collective: every rank calls it.  Each rank writes 8 rounds of 128-byte lines (flag in
 * the 8th 16 B) into its successor's LL128 area while reading the lines its predecessor
 * writes, and counts lines whose flag arrived without their data (or that never arrived
 * within the watchdog).  The counts — plus, from hvd_connect, whether NVML reports both
 * ring links as NVLink — are summed over the ranks with the LL protocol (8-byte words,
 * single-copy atomic by PTX), and a non-zero sum disables LL128 (LL128_MAX_BYTES = 0)
 * on every rank.  force_fail != 0 makes this rank report a failure (test hook; the
 * environment variable HVD_LL128_SELFTEST_FORCE_FAIL=1 does the same inside
 * hvd_connect).  *status = HVD_CFG_LL128_STATUS.  Synchronises the device.
 * Errors: INVALID, NOT_CONNECTED, CUDA; a peer that never writes makes its lines count
 * as missing (the check fails, it does not hang). */
int hvd_ll128_selftest(hvd_comm* c, int force_fail, int* status);

/* Latched asynchronous error (HVD_OK if none).  Non-blocking. */
int hvd_poll_error(hvd_comm* c);
const char* hvd_strerror(int status);

/* "hvd-src-<sha256 prefix>" of the sources this library was compiled from (the build
 * step compares it with the tree to decide whether to recompile).  Static string. */
const char* hvd_build_id(void);

/* Device-side traffic counters of local rank `local` since init: bytes pushed
 * to the successor and chunk messages sent (one per ring iteration; P:L197-198
 * "communicates with two of its peers 2*(N-1) times").  Reads device memory
 * (synchronises the device).  Errors: INVALID, CUDA. */
int hvd_traffic(hvd_comm* c, int local, uint64_t* sent_bytes, uint64_t* sends);

typedef enum {
  HVD_CFG_CHANNELS = 1,      /* CTAs per rank in the ring kernel (1..256)               */
  HVD_CFG_SLICE_BYTES = 2,   /* pipelining slice target per channel (0 = auto: half of a
                                channel's share of a chunk, 32..128 KiB); a share is cut into
                                ceil(share / target) equal slices, rounded up to 256 B     */
  HVD_CFG_THREADS = 3,       /* data threads per ring CTA (64..384, multiple of 32, default 256; +1 signal warp) */
  HVD_CFG_TIMEOUT_MS = 4,    /* device spin-wait watchdog                               */
  HVD_CFG_PACK_CTAS_PER_SM = 5,
  HVD_CFG_PROFILE = 6,       /* 1: record CUDA events around every kernel launch        */
  HVD_CFG_SIGNAL_MODE = 7,   /* ring signal: 1 fence.acq_rel.sys + relaxed store, 2 st.release.sys */
  HVD_CFG_FUSED = 8,         /* 1 (default): pack + ring + unpack in one zero-copy kernel per
                                fusion buffer; 0: three kernels (pack, ring, unpack)       */
  HVD_CFG_TIMELINE = 9,      /* > 0: record a device timeline of every fused launch with up to
                                this many slice records per channel; 0: off (default)      */
  HVD_CFG_WINDOW = 10,       /* fused: max slices per channel pushed but not yet published,
                                the one being pushed included (default 2; 0 = no limit; 1 = a slice
                                starts only after the previous one's signal is out): bounds
                                the NVLink backlog a fence waits for, so the signal latency */
  HVD_CFG_FIN_LAG = 11,      /* fused: slices by which the final local scatter trails the last
                                all-gather iteration (>= K-1: scatter after all of it)     */
  HVD_CFG_LL128_MAX_BYTES = 15, /* a call that is one fusion buffer larger than LL_MAX_BYTES
                                and of at most this many bytes uses the LL128 protocol: flags
                                inside 128-byte lines (relies on NVLink delivering a warp's
                                128 B line store whole; 16/15 wire bytes).  In a call of more
                                than 16 buffers at N > 2 (fusion off), buffers above the
                                multi-buffer LL limit and up to min(this, 16 MiB) go to
                                grouped LL128 launches.  Default 24 MiB at N = 2, 48 MiB at
                                N > 2 when every ring link is NVLink and the connect-time
                                line-atomicity self-test passed, else 0; max 64 MiB;
                                0 = never.                                                  */
  HVD_CFG_LL_MAX_BYTES = 14, /* a call that is one fusion buffer of at most this many bytes
                                (default 256 KiB; max 8 MiB; 0 = never, also in multi-buffer calls)
                                uses the LL protocol: {epoch, data} words, no fences or
                                counters (fp32/bf16/i32) */
  HVD_CFG_MULTI_BUFFERS = 13, /* fusion buffers per fused launch (1..96, default 96): the
                                buffers of one call pipeline inside one persistent launch  */
  HVD_CFG_PROTOCOL = 12,     /* allreduce data movement for buffers above the LL / LL128
                                limits: 2 bulk push — the TMA engine moves every stage
                                through shared memory (cp.async.bulk loads and stores into
                                the successor's HBM), only for calls whose tensors share the
                                wire dtype; 1 push — SM stores into the successor's HBM;
                                0 pull — each rank TMA-loads its predecessor's partials
                                (needs HVD_CFG_PULL_BUFFERS: virtual mode allocates them
                                here, a real rank returns INVALID without them).
                                Same ring order, same bits.                                 */
  HVD_CFG_BULK_STAGES = 16,  /* bulk push: shared-memory stages per CTA (2..8)                */
  HVD_CFG_BULK_STAGE_BYTES = 17, /* bulk push: bytes per stage (4 KiB..64 KiB, multiple of 1 KiB) */
  HVD_CFG_BULK_DEPTH = 18,   /* bulk push: bulk-store groups a CTA leaves incomplete before it
                                publishes a stage's op (0..3); a stage's shared memory is
                                reused as soon as its stores have read it                   */
  HVD_CFG_BULK_CHANNELS = 19, /* bulk push: CTAs per rank (1..256; capped by co-residency)  */
  HVD_CFG_BULK_SLICE_BYTES = 20, /* bulk push: signal slice per channel (multiple of 256 B) */
  HVD_CFG_SIGNAL_WARPS = 21, /* fused push: signal warps per CTA (1..4; THREADS + 32 x this
                                <= 416): each fences and publishes with a max, so fences overlap */
  HVD_CFG_LL128_STATUS = 22, /* read only (hvd_get_config): outcome of the LL128 line-atomicity
                                self-test: 0 not run (N = 1, or a virtual comm that did not
                                call hvd_ll128_selftest), 1 passed, -1 torn or missing lines,
                                -2 a ring link is not NVLink, -3 failure forced (test hook).
                                Any failure sets LL128_MAX_BYTES to 0 on every rank.        */
  HVD_CFG_SOLO_KERNEL = 23,  /* N = 1 (gather x 1/N -> scatter, an HBM stream): 0 (default)
                                one CTA per 16 KiB tile; 1 persistent bulk-copy kernel (one
                                CTA per SM streaming tiles through shared-memory stages: each
                                byte holds shared memory from load issue to store read, which
                                measured slower).  Both use programmatic dependent launch.
                                Tensors whose dtype differs from the wire dtype always take
                                the tile kernel.                                            */
  HVD_CFG_SOLO_STAGES = 24,  /* N = 1 bulk kernel: shared-memory stages per CTA (2..8)      */
  HVD_CFG_SOLO_STAGE_BYTES = 25, /* N = 1 bulk kernel: bytes per stage (4..64 KiB, x 1 KiB)  */
  HVD_CFG_PACE_GBPS = 26,    /* fused push: pace each rank's remote stores to this many GB/s,
                                split evenly over the channels (0 = unpaced).  Keeps the NVLink
                                store queue, and with it every ring hop's latency, short     */
  HVD_CFG_PACE_BURST_ROWS = 27, /* pacing credit a channel may accumulate while idle, in rows
                                of remote stores (threads x 16 B); default 2                */
  HVD_CFG_FUSED_PDL = 28,    /* fused push: programmatic dependent launch, so back-to-back calls
                                overlap the next launch with this one's tail (0 off; 1 with the
                                cooperative launch; 2 instead of it, one local rank only)   */
  HVD_CFG_WATCHER = 29,      /* fused push: 1 = a lane of the signal warp watches the
                                predecessor's counter and mirrors it in shared memory; the
                                slice loop then waits on shared memory                      */
  HVD_CFG_HOST_ZERO_COPY = 30, /* hvd_allreduce_host: 1 = when every buffer is pinned host
                                memory the device addresses directly, the ring kernels gather
                                from / scatter to it over PCIe (no staging copies); 0
                                (default) = the staged H2D / ring / D2H pipeline, measured
                                faster (64 MiB: N = 1 1.7 vs 1.9 ms, N = 4 3.9 vs 8.9 ms)   */
  HVD_CFG_PREISSUE = 31,     /* fused push: 1 = a slice that gathers the local gradient and adds
                                the received partial issues its first gradient loads before
                                waiting for the predecessor's signal; 0 = after; -1 (default)
                                = on for N > 2 (64 MiB at N = 4: 165.4 -> 162.2 us; N = 2
                                neutral)                                                   */
  HVD_CFG_LL_PDL = 32,       /* LL / LL128 launches: programmatic dependent launch (back-to-back
                                small calls overlap the next launch with this one's tail);
                                default 1 (N = 4, <= 1 MiB: 1-7 % lower latency)           */
  HVD_CFG_PULL_BUFFERS = 33, /* 1 = allocate the pull protocol's two buffers (2 x the region
                                buffer size, a separate device allocation) so that
                                HVD_CFG_PROTOCOL = 0 can be chosen.  Real ranks: set before
                                hvd_get_ipc_blob, identically on every rank (hvd_connect
                                returns INVALID otherwise); virtual mode: any time.  Default 0
                                (the environment variable HVD_PULL_BUFFERS=1 at init: 1).
                                Cannot be turned off once allocated (INVALID).              */
  HVD_CFG_SOLO_TAIL = 34     /* N = 1: the last this many member tiles of a buffer are cut in
                                half so that the final wave drains sooner (-1 = one wave,
                                9 x the SM count; 0 = off, the default).  Drops cached plans. */
} hvd_config_key;
/* Set a tuning knob; every rank must set identical values.  Errors: INVALID. */
int hvd_set_config(hvd_comm* c, int key, int64_t value);
int64_t hvd_get_config(const hvd_comm* c, int key);

typedef enum { HVD_KERNEL_PACK = 0, HVD_KERNEL_RING = 1, HVD_KERNEL_UNPACK = 2, HVD_KERNEL_SCALE = 3,
               HVD_KERNEL_FUSED = 4, HVD_KERNEL_COPY = 5, HVD_KERNEL_PULL = 6, HVD_KERNEL_LL = 7,
               HVD_KERNEL_SOLO = 8, HVD_KERNEL_LL128 = 9, HVD_KERNEL_BULK = 10,
               HVD_KERNEL_KINDS = 11 } hvd_kernel_kind;
/* Kernel launches of each kind since the last call (always counted) and, with
 * HVD_CFG_PROFILE on, the summed device time in ms between the CUDA events
 * recorded on the launch stream around each launch (waits for those events).
 * launches[HVD_KERNEL_KINDS], device_ms[HVD_KERNEL_KINDS]; counters reset.
 * Errors: INVALID, CUDA. */
int hvd_kernel_stats(hvd_comm* c, uint64_t* launches, double* device_ms);

/* Horovod Timeline ("view exactly what each node was doing at each time
 * step"), recorded on the device: with HVD_CFG_TIMELINE on, the most recent fused
 * launch of local rank `local` leaves, per channel, `slices` data records
 * {t_begin, t_end} (ns, %globaltimer) of its slice operations in program order
 * (iteration t = index / K: reduce-scatter t < N-1, all-gather after, the final
 * local scatter last) followed, at word offset channels_max * words_per_channel,
 * by `signals` records {t_publish, slices_published} of its signal warp.
 * out == NULL returns only `info`; otherwise cap_words must be >= the buffer
 * size (256 * words_per_channel * 2).  Synchronises the device.  Errors: INVALID. */
typedef struct {
  int32_t channels, slices, signals, K, T, rank, size;
  int32_t kind;  /* 0: fused push kernel (T = 2(N-1) iterations + final scatter; signal records)
                    1: pull kernel (T = 2N-1 steps, op j = t*K + k in order; the second record
                       array holds {t_loadable, op} of the loader warp)                       */
  uint64_t words_per_channel;
} hvd_timeline_info;
int hvd_timeline(hvd_comm* c, int local, uint64_t* out, uint64_t cap_words, hvd_timeline_info* info);

/* Job-wide Horovod Timeline ("view exactly what each node was doing at each
 * time step throughout a training job"; "enable timelines by setting a single environment
 * variable").  HVD_TIMELINE=<path> in the environment turns it on for every
 * comm at hvd_init (single process / virtual) or hvd_connect (multi-process); these
 * calls do the same programmatically.  Output: Chrome trace-event JSON (about:tracing /
 * chrome://tracing), an array written incrementally, one event per line, without the
 * closing bracket (Chrome accepts it; a crashed job keeps its trace).  Per rank (pid):
 *   tid 0 "host calls":     one "X" span per public call (ALLREDUCE, ALLREDUCE_BUFFER,
 *                           ALLREDUCE_HOST, NEGOTIATE_ALLREDUCE, BROADCAST, ALLGATHER),
 *                           args {call, tensors, bytes, launches, status};
 *   tid 1 "device kernels": one "X" span per kernel launch (FUSED_RING, LL_RING,
 *                           LL128_RING, BULK_RING, PULL_RING, COPY_RING, SOLO, PACK, RING,
 *                           UNPACK, SCALE) from its first CTA's start to its last CTA's
 *                           end on that rank's GPU, args {seq, call, ctas, bytes};
 *   tid 2 "negotiation":    one "X" span per tensor agreed by hvd_allreduce_negotiated, from
 *                           its ready report to the cycle that agreed it, args {tensor, call};
 *   "s"/"f" flow events link each call to its launches.
 * Device times are %globaltimer converted to CLOCK_REALTIME (offset calibrated at start,
 * uncertainty in the TIMELINE_START event), so the ranks of a node share one time axis.
 * Every rank appends to the same file (O_APPEND, whole lines per write).  Records of
 * finished launches are written at every call and by hvd_timeline_flush without a
 * device synchronisation; hvd_timeline_stop / hvd_finalize synchronise and write the rest.
 *
 * hvd_timeline_start: path = trace file; truncate != 0 starts a new file (one rank of a
 *   job; the others must start after it).  Errors: INVALID (already on, bad path), CUDA.
 * hvd_timeline_stop:  synchronises the device, writes every record, closes.  Errors: CUDA.
 * hvd_timeline_flush: writes the records of finished launches (non-blocking); *launches /
 *   *dropped (either may be NULL) = launches traced / records lost (never finished, or
 *   overwritten before being written: more than 4096 launches outstanding).           */
int hvd_timeline_start(hvd_comm* c, const char* path, int truncate);
int hvd_timeline_stop(hvd_comm* c);
int hvd_timeline_flush(hvd_comm* c, uint64_t* launches, uint64_t* dropped);

/* ---- host-only plan inspection (no device needed) -------------------------------------------- */

typedef struct {
  int32_t tensor;    /* index into the submitted list */
  int32_t buffer;    /* fusion buffer index */
  uint64_t src_off;  /* element offset in the tensor */
  uint64_t dst_off;  /* element offset in the fusion buffer */
  uint64_t count;    /* elements */
} hvd_plan_entry;

typedef struct {
  int32_t dtype;
  int32_t n_entries;
  int32_t first_entry;
  int32_t reserved;
  uint64_t length;   /* L, elements */
} hvd_plan_buffer;

/* Compute the Tensor Fusion plan of (counts[k], dtypes[k]) exactly as
 * hvd_allreduce does.  On input *n_entries / *n_buffers are the capacities of
 * the output arrays; on output the sizes used.  Errors: INVALID (capacity too
 * small: sizes needed are returned), UNSUPPORTED (dtype). */
int hvd_plan(const uint64_t* counts, const int32_t* dtypes, int n, uint64_t fusion_threshold,
             uint64_t capacity, hvd_plan_entry* entries, int* n_entries, hvd_plan_buffer* buffers,
             int* n_buffers);

/* Chunk partition of a buffer of `length` elements over `size` ranks
 * ("chunks of the data buffer"; R2): out[0..size] boundaries. */
int hvd_chunk_bounds(uint64_t length, int size, int dtype, uint64_t* out);

/* Allreduce of `count` elements held in HOST memory (pinned for overlap):
 * in[l] -> out[l] for each local rank l (in and out may alias).  The buffer is
 * cut into chunks of `chunk_bytes` (0 = 8 MiB); chunk i is copied to the device
 * on one copy stream, reduced on `stream` exactly as hvd_allreduce reduces one
 * tensor (so same bits), and copied back on another copy stream while chunk
 * i+1 is copied in: PCIe in, the ring and PCIe out overlap (3 device staging
 * slots, library-owned).  When every in / out buffer is pinned host memory the device
 * addresses at the same pointer (UVA; e.g. cudaHostAlloc, torch pin_memory) and
 * HVD_CFG_HOST_ZERO_COPY is on (default off), there is no staging: the call is hvd_allreduce
 * of one tensor whose gather reads `in` and whose scatter writes `out` over PCIe inside
 * the ring kernels (same bits, same traffic: count elements each way; chunk_bytes is
 * ignored).  Completion: `stream`.  Host buffers must stay valid until then.
 * Errors: INVALID, UNSUPPORTED (dtype / AVERAGE on integers), CUDA. */
int hvd_allreduce_host(hvd_comm* c, const void* const* in, void* const* out, uint64_t count, int dtype, int op,
                       uint64_t chunk_bytes, void* stream);

/* ---------------------------------------------------------------- readiness negotiation
 * Tensor Fusion step 1, "Determine which tensors are ready to be reduced" and
 * step 6, "Repeat until there are no more tensors to reduce in the cycle"
 * (P:L366).  The paper does not say how ranks agree on readiness;
 * DESIGN.md R15 takes SPEC's reading: a tensor is globally ready
 * when every rank has reported it; globally ready tensors are reduced in rank
 * 0's submission order; the others stay pending for a later cycle.
 *
 * Host-only control plane (no GPU needed).  Tensors are named by dense ids
 * 0..max_tensors-1 (e.g. registration order).  Ranks of one node share a POSIX
 * shared-memory segment `shm_name` ("/name"; created by rank 0, opened by the
 * others, retried until it exists): per rank and cycle parity, the ordered
 * pending list {id, dtype, count}.  A cycle publishes this process's lists, waits
 * until every rank has published the same cycle, and intersects — every rank
 * computes the same answer, so no coordinator round trip is needed.  Parities
 * alternate: a rank cannot overwrite cycle k's list before every rank has
 * finished reading it (it must first see all ranks publish cycle k+1).
 * shm_name == NULL: process-private segment for `nlocal` ranks rank..rank+nlocal-1
 * of a virtual communicator (hvd_init_virtual); otherwise nlocal must be 1. */
typedef struct hvd_negotiator hvd_negotiator;
/* Errors: INVALID (arguments), TIMEOUT (segment never appeared), UNSUPPORTED (shm). */
int hvd_negotiator_create(const char* shm_name, int rank, int size, int nlocal, uint32_t max_tensors,
                          uint64_t timeout_ms, hvd_negotiator** out);
/* Mark tensor `id` ready on local rank `local` (count elements of dtype); it joins
 * the end of that rank's pending list.  Errors: INVALID (id out of range, already
 * pending, bad dtype). */
int hvd_negotiator_ready(hvd_negotiator* g, int local, uint32_t id, uint64_t count, int dtype);
/* One negotiation cycle (collective over all ranks): ids_out[0..*n_out) = the
 * globally ready ids in rank 0's submission order, removed from every rank's
 * pending list.  ids_out has room for max_tensors ids.  Errors: TIMEOUT (a rank
 * did not publish within timeout_ms), INVALID (the same id reported with a
 * different dtype or count by two ranks: the protocol error of S:L299; the id is
 * returned in *n_out). */
int hvd_negotiator_cycle(hvd_negotiator* g, uint32_t* ids_out, uint32_t* n_out);
/* Pending ids of local rank `local` (in submission order; ids_out may be NULL). */
int hvd_negotiator_pending(const hvd_negotiator* g, int local, uint32_t* ids_out, uint32_t* n_out);
/* Negotiation records for the Horovod Timeline (P:L326-349 shows each tensor's
 * negotiation phase): for every id agreed since the last read, out[3i..3i+2] =
 * {id, ns when local rank `local` reported it ready, ns when the cycle agreed
 * it} (CLOCK_REALTIME, comparable across the processes of a node).  out = NULL:
 * *n_out = records available.  Records read are dropped.  Errors: INVALID. */
int hvd_negotiator_trace(hvd_negotiator* g, int local, uint64_t* out, uint32_t cap, uint32_t* n_out);
/* Unmap (rank 0 also unlinks the segment).  Idempotent on NULL. */
int hvd_negotiator_destroy(hvd_negotiator* g);

/* One cycle, then the allreduce of the agreed tensors (P:L366-373 in full):
 * tensors[l * n + id] is local rank l's tensor `id` (n = the id space used);
 * the agreed ids (ids_out, capacity n) are reduced in that order through the
 * same Tensor Fusion plan and ring as hvd_allreduce.  Errors: those of
 * hvd_negotiator_cycle and hvd_allreduce; INVALID if an agreed tensor's count or
 * dtype differs from what was reported ready. */
int hvd_allreduce_negotiated(hvd_comm* c, hvd_negotiator* g, const hvd_tensor* tensors, uint32_t n, int op,
                             uint64_t fusion_threshold, void* stream, uint32_t* ids_out, uint32_t* n_out);

#ifdef __cplusplus
}
#endif
#endif /* HVD_B200_H */

"""CPU oracle for the fused ring allreduce of Horovod (arXiv 1802.05799).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product path (``paper_1802_05799_b200``) never imports it and
shares no code with it.

It is a plain, slow, obviously-correct numpy simulation of N ranks that
runs the paper's algorithm step by step, in the paper's order:

  Tensor Fusion (§7)
    1. "Select the first few tensors that fit in the buffer and have the
       same data type"                         -> ``fusion_plan``
    2. "Allocate a fusion buffer ... 64 MB"    -> ``DEFAULT_FUSION_BYTES``
    3. "Copy data of selected tensors into the fusion buffer" -> ``pack``
       (fused with the averaging 1/N of P:L143, reading R1)
    4. "Execute the allreduce operation on the fusion buffer" -> ``ring_allreduce``
    5. "Copy data from the fusion buffer into the output tensors" -> ``unpack``
    6. "Repeat until there are no more tensors"  -> loop in ``allreduce``

  Ring-allreduce (§3)
    "each of N nodes communicates with two of its peers 2*(N-1) times ...
     In the first N-1 iterations, received values are added to the values
     in the node's buffer. In the second N-1 iterations, received values
     replace the values held in the node's buffer."
    Schedule (reading R3, after Patarasuk & Yuan):
    rank r sends to r+1; in reduce-scatter step s it sends chunk (r-s) mod N,
    in all-gather step s it sends chunk (r+1-s) mod N.

Readings of silent/ambiguous passages are listed in DESIGN.md §Readings
(R1..R14); the ones this file implements are cited inline.

Value representation: see ``workloads`` (bf16 = uint16 bit patterns).
Parity pins for every function live in ``tests/test_oracle_pins.py``.
Parity unpinned (conventions with no paper value): the chunk quantum
(256 B), the 16 B member alignment and the oversized-tensor split rule.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

DEFAULT_FUSION_BYTES = 64 * 1024 * 1024  # P:L368-369 "Default fusion buffer size is 64 MB" (R9)
MEMBER_ALIGN_BYTES = 16                   # R2: member offsets aligned to 16 B (convention)
CHUNK_QUANTUM_BYTES = 256                 # R2: chunk boundaries on 256 B (convention)

ELEM_SIZE = {"f32": 4, "bf16": 2, "i32": 4, "i64": 8}
NP_TYPE = {"f32": np.float32, "bf16": np.uint16, "i32": np.int32, "i64": np.int64}
FLOAT_TYPES = ("f32", "bf16")


# --------------------------------------------------------------------------
# bfloat16 helpers (R4): bf16 is the top half of an IEEE binary32.
# --------------------------------------------------------------------------
def bf16_to_f32(h: np.ndarray) -> np.ndarray:
    """Exact widening: the bf16 bits become the high 16 bits of a binary32."""
    return (h.astype(np.uint32) << np.uint32(16)).view(np.float32)


def f32_to_bf16_rne(x: np.ndarray) -> np.ndarray:
    """Round binary32 to bfloat16, round-to-nearest-even, on the bits.

    u' = u + 0x7FFF + ((u >> 16) & 1); result = u' >> 16.  NaN maps to a
    quiet NaN of the same sign (R10: NaN is compared by class only).
    """
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    lsb = (u >> np.uint32(16)) & np.uint32(1)
    r = ((u + np.uint32(0x7FFF) + lsb) >> np.uint32(16)).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        r = r.copy()
        r[nan] = ((u[nan] >> np.uint32(16)) | np.uint32(0x0040)).astype(np.uint16)
    return r


# --------------------------------------------------------------------------
# Elementwise arithmetic of the wire dtype (R4, R11)
# --------------------------------------------------------------------------
def add_w(a: np.ndarray, b: np.ndarray, dtype: str) -> np.ndarray:
    """One reduction add as the paper's step "received values are added"."""
    with np.errstate(all="ignore"):
        if dtype == "f32":
            return (a + b).astype(np.float32)            # binary32 RN add
        if dtype == "bf16":
            return f32_to_bf16_rne(bf16_to_f32(a) + bf16_to_f32(b))  # fp32 add, RNE to bf16
        return (a + b).astype(NP_TYPE[dtype])        # two's-complement wrap (R11)


def scale_w(x: np.ndarray, s: np.float32, dtype: str) -> np.ndarray:
    """Averaging prescale (R1): fl32(x * s), then cast to the wire dtype."""
    with np.errstate(all="ignore"):
        if dtype == "f32":
            return (x * s).astype(np.float32)
        if dtype == "bf16":
            return f32_to_bf16_rne(bf16_to_f32(x) * s)
    raise ValueError("AVERAGE is undefined for integer dtypes (R11)")


def to_wire(x: np.ndarray, dtype: str, wire: str, s) -> np.ndarray:
    """Pack with a wire dtype: fl32(f32(x) * s), then cast to ``wire``.

    ``s`` is None for SUM.  f32 -> bf16 wire rounds RNE; bf16 -> f32 wire widens exactly.
    """
    with np.errstate(all="ignore"):
        f = bf16_to_f32(x) if dtype == "bf16" else np.asarray(x, dtype=np.float32)
        if s is not None:
            f = (f * s).astype(np.float32)
        return f32_to_bf16_rne(f) if wire == "bf16" else f.astype(np.float32)


def from_wire(b: np.ndarray, wire: str, dtype: str) -> np.ndarray:
    """Unpack with a wire dtype: bf16 wire -> f32 widens exactly; f32 wire -> bf16 rounds RNE."""
    if wire == dtype:
        return b
    return bf16_to_f32(b) if wire == "bf16" else f32_to_bf16_rne(b)


def inv_n(nranks: int) -> np.float32:
    """s = fl32(1/N) (R1)."""
    return np.float32(1.0) / np.float32(nranks)


# --------------------------------------------------------------------------
# Tensor Fusion plan (§7 step 1; R6, R7, R8)
# --------------------------------------------------------------------------
@dataclass
class Entry:
    tensor: int      # index into the submitted list
    src_off: int     # element offset inside the tensor
    dst_off: int     # element offset inside the fusion buffer
    count: int       # elements


@dataclass
class FusionBuffer:
    dtype: str
    entries: list = field(default_factory=list)
    length: int = 0  # L, elements (end of the last member)


def _align_up(v: int, a: int) -> int:
    return (v + a - 1) // a * a


def fusion_plan(tensors, threshold: int = DEFAULT_FUSION_BYTES,
                capacity: int = DEFAULT_FUSION_BYTES):
    """Next-fit fusion in submission order.

    ``tensors`` is a list of (count, dtype).  "Select the first few tensors
    that fit in the buffer and have the same data type": a
    tensor joins the open buffer when the dtype matches and its 16 B aligned
    offset plus its bytes is <= the limit ("fits", inclusive: R6); otherwise
    the open buffer is closed and a new one opened.  ``threshold == 0`` turns
    fusion off: every tensor is its own buffer (R8).  The limit is
    ``min(threshold, capacity)`` (or ``capacity`` when fusion is off); a
    tensor larger than the limit is split into segments of
    floor(limit/esz) elements, each a singleton buffer (R7).  Tensors with
    zero elements are skipped.
    """
    limit = capacity if threshold == 0 else min(threshold, capacity)
    out = []
    cur = None
    for k, (count, dtype) in enumerate(tensors):
        if count == 0:
            continue
        esz = ELEM_SIZE[dtype]
        nbytes = count * esz
        if nbytes > limit:
            if cur is not None:
                out.append(cur)
                cur = None
            seg = limit // esz
            for start in range(0, count, seg):
                n = min(seg, count - start)
                out.append(FusionBuffer(dtype, [Entry(k, start, 0, n)], n))
            continue
        if threshold == 0:
            out.append(FusionBuffer(dtype, [Entry(k, 0, 0, count)], count))
            continue
        if cur is not None and cur.dtype == dtype:
            off_bytes = _align_up(cur.length * esz, MEMBER_ALIGN_BYTES)
            if off_bytes + nbytes <= limit:
                off = off_bytes // esz
                cur.entries.append(Entry(k, 0, off, count))
                cur.length = off + count
                continue
        if cur is not None:
            out.append(cur)
        cur = FusionBuffer(dtype, [Entry(k, 0, 0, count)], count)
    if cur is not None:
        out.append(cur)
    return out


# --------------------------------------------------------------------------
# Chunk partition ("chunks of the data buffer"; R2)
# --------------------------------------------------------------------------
def chunk_bounds(length: int, nranks: int, dtype: str):
    """Boundaries b[0..N] of the N chunks of a buffer of ``length`` elements.

    q = ceil(L / (N*g)) * g with g = 256 B in elements; chunk c is
    [min(c*q, L), min((c+1)*q, L)) (R2).
    """
    g = CHUNK_QUANTUM_BYTES // ELEM_SIZE[dtype]
    q = -(-length // (nranks * g)) * g
    return [min(c * q, length) for c in range(nranks)] + [length]


# --------------------------------------------------------------------------
# Pack / unpack (§7 steps 3 and 5)
# --------------------------------------------------------------------------
def pack(xs, fb: FusionBuffer, scale):
    """buf[dst+i] = cvt_w(fl32(x_k[src+i] * s)); interior padding is zero.

    ``scale`` is None for SUM (plain copy) or fl32(1/N) for AVERAGE (R1).
    """
    buf = np.zeros(fb.length, dtype=NP_TYPE[fb.dtype])
    for e in fb.entries:
        x = xs[e.tensor][e.src_off:e.src_off + e.count]
        buf[e.dst_off:e.dst_off + e.count] = x if scale is None else scale_w(x, scale, fb.dtype)
    return buf


def unpack(buf, fb: FusionBuffer, outs):
    """x_k[src+i] = buf[dst+i] (in place into ``outs``)."""
    for e in fb.entries:
        outs[e.tensor][e.src_off:e.src_off + e.count] = buf[e.dst_off:e.dst_off + e.count]


# --------------------------------------------------------------------------
# Ring allreduce over N simulated ranks (§3; R3)
# --------------------------------------------------------------------------
@dataclass
class Traffic:
    sends: int = 0          # number of chunk messages sent
    sent_elems: int = 0     # elements sent
    recv_elems: int = 0     # elements received


def ring_allreduce(bufs, dtype: str, traffic=None):
    """Run the 2(N-1) ring iterations on the N rank buffers, in place.

    Reduce-scatter, s = 0..N-2: every rank r sends chunk (r-s) mod N to
    r+1; the receiver adds it into its own copy ("received values are
    added").  All-gather, s = 0..N-2: rank r sends chunk (r+1-s) mod N to
    r+1; the receiver overwrites ("received values replace").  Messages of a
    step are snapshotted before any rank applies them, i.e. all sends of an
    iteration happen concurrently.
    """
    n = len(bufs)
    if traffic is None:
        traffic = [Traffic() for _ in range(n)]
    if n == 1:
        return bufs, traffic
    b = chunk_bounds(len(bufs[0]), n, dtype)

    def sl(c):
        return slice(b[c], b[c + 1])

    for s in range(n - 1):                      # first N-1 iterations: add
        msgs = [bufs[r][sl((r - s) % n)].copy() for r in range(n)]
        for r in range(n):
            c = (r - 1 - s) % n                 # chunk sent by r-1 this step
            m = msgs[(r - 1) % n]
            bufs[r][sl(c)] = add_w(bufs[r][sl(c)], m, dtype)
            traffic[(r - 1) % n].sends += 1
            traffic[(r - 1) % n].sent_elems += len(m)
            traffic[r].recv_elems += len(m)
    for s in range(n - 1):                      # second N-1 iterations: replace
        msgs = [bufs[r][sl((r + 1 - s) % n)].copy() for r in range(n)]
        for r in range(n):
            c = (r - s) % n
            m = msgs[(r - 1) % n]
            bufs[r][sl(c)] = m
            traffic[(r - 1) % n].sends += 1
            traffic[(r - 1) % n].sent_elems += len(m)
            traffic[r].recv_elems += len(m)
    return bufs, traffic


# --------------------------------------------------------------------------
# The whole hot path: allreduce(-average) of a tensor list
# --------------------------------------------------------------------------
def allreduce(xs_by_rank, dtypes, op: str = "average",
              threshold: int = DEFAULT_FUSION_BYTES,
              capacity: int = DEFAULT_FUSION_BYTES, wire=None):
    """Tensor Fusion steps 1-6 around the ring, for every simulated rank.

    ``xs_by_rank[r][k]`` is tensor k on rank r (numpy, ``workloads`` format),
    ``dtypes[k]`` its dtype.  ``op`` is "sum" or "average".
    ``wire`` (R14): the fusion buffer / ring dtype when it differs from the
    tensors' (all tensors must then share one float dtype); None = same.
    Returns (outs_by_rank, traffic_per_rank, plan).
    """
    n = len(xs_by_rank)
    counts = [len(x) for x in xs_by_rank[0]]
    if wire is not None and any(d != wire for d in dtypes):
        if len(set(dtypes)) != 1 or dtypes[0] not in FLOAT_TYPES or wire not in FLOAT_TYPES:
            raise ValueError("a wire dtype needs one float tensor dtype (R14)")
        tdt = dtypes[0]
        plan = fusion_plan([(c, wire) for c in counts], threshold, capacity)
        outs = [[x.copy() for x in xs] for xs in xs_by_rank]
        traffic = [Traffic() for _ in range(n)]
        scale = inv_n(n) if op == "average" else None
        for fb in plan:
            bufs = []
            for r in range(n):
                buf = np.zeros(fb.length, dtype=NP_TYPE[wire])
                for e in fb.entries:
                    x = xs_by_rank[r][e.tensor][e.src_off:e.src_off + e.count]
                    buf[e.dst_off:e.dst_off + e.count] = to_wire(x, tdt, wire, scale)
                bufs.append(buf)
            ring_allreduce(bufs, wire, traffic)
            for r in range(n):
                for e in fb.entries:
                    outs[r][e.tensor][e.src_off:e.src_off + e.count] = from_wire(
                        bufs[r][e.dst_off:e.dst_off + e.count], wire, tdt)
        return outs, traffic, plan
    plan = fusion_plan(list(zip(counts, dtypes)), threshold, capacity)
    outs = [[x.copy() for x in xs] for xs in xs_by_rank]
    traffic = [Traffic() for _ in range(n)]
    for fb in plan:                                       # step 6: repeat
        if op == "average" and fb.dtype not in FLOAT_TYPES:
            raise ValueError("AVERAGE is undefined for integer dtypes (R11)")
        scale = inv_n(n) if op == "average" else None
        bufs = [pack(xs_by_rank[r], fb, scale) for r in range(n)]      # step 3
        ring_allreduce(bufs, fb.dtype, traffic)                       # step 4
        for r in range(n):
            unpack(bufs[r], fb, outs[r])                              # step 5
    return outs, traffic, plan


def allreduce_buffer(bufs, dtype: str, op: str = "sum"):
    """Raw ring on one (already packed) buffer per rank; AVERAGE prescales."""
    n = len(bufs)
    if op == "average":
        bufs = [scale_w(b, inv_n(n), dtype) for b in bufs]
    else:
        bufs = [b.copy() for b in bufs]
    return ring_allreduce(bufs, dtype)


# --------------------------------------------------------------------------
# Broadcast (§4 item 4) and allgather (north_star; R12)
# --------------------------------------------------------------------------
def broadcast(xs_by_rank, root: int):
    """Pipelined ring forward from ``root``: root -> root+1 -> ... -> root-1.

    Each non-root rank receives the root's data once and every rank except
    root-1 forwards it; results are bitwise copies of the root's input.
    """
    n = len(xs_by_rank)
    traffic = [Traffic() for _ in range(n)]
    outs = [[x.copy() for x in xs] for xs in xs_by_rank]
    for hop in range(n - 1):
        src = (root + hop) % n
        dst = (src + 1) % n
        for k, x in enumerate(outs[src]):
            outs[dst][k] = x.copy()
            traffic[src].sends += 1
            traffic[src].sent_elems += len(x)
            traffic[dst].recv_elems += len(x)
    return outs, traffic


def allgather(xs_by_rank):
    """Ring all-gather of one equal-length block per rank (R12).

    Step s = 0..N-2: rank r sends block (r-s) mod N to r+1.  The output on
    every rank is the concatenation of the blocks in rank order.
    """
    n = len(xs_by_rank)
    count = len(xs_by_rank[0])
    traffic = [Traffic() for _ in range(n)]
    outs = []
    for r in range(n):
        o = np.zeros(n * count, dtype=xs_by_rank[r].dtype)
        o[r * count:(r + 1) * count] = xs_by_rank[r]
        outs.append(o)
    for s in range(n - 1):
        msgs = [outs[r][((r - s) % n) * count:((r - s) % n + 1) * count].copy() for r in range(n)]
        for r in range(n):
            blk = (r - 1 - s) % n
            outs[r][blk * count:(blk + 1) * count] = msgs[(r - 1) % n]
            traffic[(r - 1) % n].sends += 1
            traffic[(r - 1) % n].sent_elems += count
            traffic[r].recv_elems += count
    return outs, traffic

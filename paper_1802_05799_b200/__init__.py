"""B200-native fused ring allreduce (Horovod, arXiv 1802.05799) — Python API.

A thin layer over the C ABI (``include/hvd.h``, ``libhvd_b200.so``): it takes
``data_ptr()`` / ``numel()`` / dtype from torch tensors, the current CUDA
stream, and exchanges CUDA-IPC blobs over a ``torch.distributed`` gloo group
at init.  Every step of the hot path (pack, ring, unpack) runs in the
library's sm_100a kernels; there is no CPU or eager-torch fallback.

The paper's user-facing calls:
    hvd.init()                              -> ``init()``
    hvd.DistributedOptimizer (averaging)    -> ``Comm.allreduce_average(grads)``
    hvd.broadcast_global_variables(0)       -> ``Comm.broadcast(tensors, root=0)``
plus ``Comm.allgather`` (north_star).  Also: ``Comm.register`` (zero-copy
gradients), ``Comm.allreduce(..., wire="bf16")`` (wire dtype, R14),
``negotiator`` / ``Comm.allreduce_negotiated`` (readiness cycle),
``Comm.allreduce_host`` (pinned host gradients), the job-wide Horovod Timeline
(``HVD_TIMELINE=<path>`` or ``Comm.timeline_start``; read back with
``timeline.load_trace``) and the per-slice ring detail of one launch (``Comm.timeline``,
``timeline.write_chrome_trace``).
"""
from __future__ import annotations

import ctypes as C
import os

from . import _lib
from ._lib import (HVD_AVERAGE, HVD_BFLOAT16, HVD_FLOAT32, HVD_INT32, HVD_INT64, HVD_SUM,  # noqa: F401
                   HvdError, check, lib)

DEFAULT_FUSION_BYTES = 64 * 1024 * 1024

_TORCH_DTYPE_CODE = None


def _dtype_code(t) -> int:
    global _TORCH_DTYPE_CODE
    if _TORCH_DTYPE_CODE is None:
        import torch
        _TORCH_DTYPE_CODE = {torch.float32: HVD_FLOAT32, torch.bfloat16: HVD_BFLOAT16,
                             torch.int32: HVD_INT32, torch.int64: HVD_INT64}
    try:
        return _TORCH_DTYPE_CODE[t.dtype]
    except KeyError:
        raise HvdError(_lib.HVD_ERR_UNSUPPORTED, f"dtype {t.dtype}") from None


def _tensor_array(tensors):
    arr = (_lib.hvd_tensor * max(1, len(tensors)))()
    for i, t in enumerate(tensors):
        if not t.is_contiguous():
            raise HvdError(_lib.HVD_ERR_INVALID, "tensors must be contiguous")
        cnt = t.numel()
        arr[i].data = t.data_ptr() if cnt else None
        arr[i].count = cnt
        arr[i].dtype = _dtype_code(t)
    return arr


_RAW_STREAM = None


def _stream_handle(stream):
    """The caller's stream (default: torch's current stream on the current device)."""
    global _RAW_STREAM
    if stream is not None:
        return C.c_void_p(stream.cuda_stream)
    if _RAW_STREAM is None:
        import torch
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)  # ~0.3 us vs ~3 us for current_stream()
        _RAW_STREAM = (lambda: raw(torch.cuda.current_device())) if raw else \
            (lambda: torch.cuda.current_stream().cuda_stream)
    return C.c_void_p(_RAW_STREAM())


_OPS = {"sum": HVD_SUM, "average": HVD_AVERAGE}


class Prepared:
    """A tensor list marshalled once (``Comm.prepare``): a training loop reduces the
    same gradient tensors every step, so the ctypes descriptor array is reused and a
    call costs one C call instead of a Python walk over hundreds of tensors."""

    def __init__(self, comm, tensors):
        flat, n = comm._flat(tensors)
        self.tensors = tensors
        self._keep = flat          # keep the storage alive
        self.arr = _tensor_array(flat)
        self.n = n


class Registered:
    """A tensor list registered with ``Comm.register`` (zero-copy both ways)."""

    def __init__(self, comm, tensors, reg_id):
        self.comm = comm
        self.tensors = tensors
        self.reg_id = reg_id


class Comm:
    """One communicator: a real ring rank, or all N ranks simulated on one GPU."""

    def __init__(self, handle: C.c_void_p, device: int):
        self._h = handle
        self.device = device

    # ---------------------------------------------------------------- identity
    @property
    def rank(self) -> int:
        return lib.hvd_rank(self._h)

    @property
    def size(self) -> int:
        return lib.hvd_size(self._h)

    @property
    def local_ranks(self) -> int:
        return lib.hvd_local_ranks(self._h)

    # ---------------------------------------------------------------- collectives
    def _flat(self, tensors):
        """Accept a list (1 local rank) or a list of per-rank lists (virtual)."""
        if self.local_ranks == 1:
            if tensors and isinstance(tensors[0], (list, tuple)):
                tensors = tensors[0]
            return list(tensors), len(tensors)
        if len(tensors) != self.local_ranks:
            raise HvdError(_lib.HVD_ERR_INVALID, "virtual comm needs one tensor list per rank")
        n = len(tensors[0])
        flat = [t for per_rank in tensors for t in per_rank]
        return flat, n

    def register(self, tensors, group=None) -> Registered:
        """Register a tensor list once (collective): later allreduces write the final values
        straight into the successor's tensors (``hvd_register``)."""
        flat, n = self._flat(tensors)
        arr = _tensor_array(flat)
        rid = C.c_int(-1)
        if self.local_ranks == 1 and self.size > 1:
            ln = C.c_uint64(0)
            check(lib.hvd_register_blob(self._h, arr, n, None, C.byref(ln)), "hvd_register_blob")
            buf = C.create_string_buffer(ln.value)
            check(lib.hvd_register_blob(self._h, arr, n, buf, C.byref(ln)), "hvd_register_blob")
            blobs = b"".join(exchange_blobs(bytes(buf.raw), group))
            check(lib.hvd_register(self._h, arr, n, blobs, ln.value, C.byref(rid)), "hvd_register")
        else:
            check(lib.hvd_register(self._h, arr, n, None, 0, C.byref(rid)), "hvd_register")
        return Registered(self, tensors, rid.value)

    def deregister(self, reg: Registered):
        check(lib.hvd_deregister(self._h, reg.reg_id), "hvd_deregister")

    def prepare(self, tensors) -> Prepared:
        """Marshal a tensor list once for repeated collectives on the same tensors."""
        return Prepared(self, tensors)

    def _marshal(self, tensors):
        if isinstance(tensors, Prepared):
            return tensors.arr, tensors.n
        flat, n = self._flat(tensors)
        return _tensor_array(flat), n

    def allreduce(self, tensors, op: str = "average", fusion_threshold: int = DEFAULT_FUSION_BYTES,
                  stream=None, wire=None):
        """In-place allreduce of the tensor list (Tensor Fusion + ring).

        ``tensors``: a list (or per-rank lists on a virtual comm) or a ``Prepared``.
        ``wire`` ("f32" / "bf16" / a torch dtype): the ring dtype when it should
        differ from the tensors' (``hvd_allreduce_ex``, R14).
        """
        if isinstance(tensors, Registered):
            if wire is not None:
                raise HvdError(_lib.HVD_ERR_UNSUPPORTED, "wire dtype with registered tensors")
            check(lib.hvd_allreduce_registered(self._h, tensors.reg_id, _OPS[op], int(fusion_threshold),
                                               _stream_handle(stream)), "hvd_allreduce_registered")
            return tensors.tensors
        arr, n = self._marshal(tensors)
        if wire is None:
            check(lib.hvd_allreduce(self._h, arr, n, _OPS[op], int(fusion_threshold), _stream_handle(stream)),
                  "hvd_allreduce")
        else:
            code = _DT_CODE[wire] if isinstance(wire, str) else _dtype_code(__import__("torch").empty((), dtype=wire))
            check(lib.hvd_allreduce_ex(self._h, arr, n, _OPS[op], int(fusion_threshold), code,
                                       _stream_handle(stream)), "hvd_allreduce_ex")
        return tensors

    def allreduce_average(self, tensors, fusion_threshold: int = DEFAULT_FUSION_BYTES, stream=None):
        """The paper's gradient averaging."""
        if isinstance(tensors, Registered):
            return self.allreduce(tensors, "average", fusion_threshold, stream)
        arr, n = self._marshal(tensors)
        check(lib.hvd_allreduce_average(self._h, arr, n, int(fusion_threshold), _stream_handle(stream)),
              "hvd_allreduce_average")
        return tensors

    def allreduce_negotiated(self, neg: "Negotiator", tensors, op: str = "average",
                             fusion_threshold: int = DEFAULT_FUSION_BYTES, stream=None):
        """One negotiation cycle, then the allreduce of the tensors ready on every rank
        (P:L366-373).  ``tensors``: indexed by id (a virtual comm: per-rank lists); returns
        the ids reduced, in order."""
        arr, n = self._marshal(tensors)
        ids = (C.c_uint32 * max(1, n))()
        m = C.c_uint32(0)
        check(lib.hvd_allreduce_negotiated(self._h, neg._h, arr, n, _OPS[op], int(fusion_threshold),
                                           _stream_handle(stream), ids, C.byref(m)), "hvd_allreduce_negotiated")
        return list(ids[:m.value])

    def allreduce_host(self, inputs, outputs=None, op: str = "average", chunk_bytes: int = 0, stream=None):
        """Allreduce of HOST tensors (pinned CPU tensors for overlap; one per local rank on a virtual
        comm): chunked H2D -> ring -> D2H, pipelined (``hvd_allreduce_host``).  In place when
        ``outputs`` is None.  Completes on ``stream``."""
        ins = list(inputs) if isinstance(inputs, (list, tuple)) else [inputs]
        outs = ins if outputs is None else (list(outputs) if isinstance(outputs, (list, tuple)) else [outputs])
        if len(ins) != self.local_ranks or len(outs) != self.local_ranks:
            raise HvdError(_lib.HVD_ERR_INVALID, "one host tensor per local rank")
        for x in ins + outs:
            if x.device.type != "cpu" or not x.is_contiguous():
                raise HvdError(_lib.HVD_ERR_INVALID, "host tensors must be contiguous CPU tensors")
        n, code = ins[0].numel(), _dtype_code(ins[0])
        pin = (C.c_void_p * len(ins))(*[x.data_ptr() for x in ins])
        pout = (C.c_void_p * len(outs))(*[x.data_ptr() for x in outs])
        check(lib.hvd_allreduce_host(self._h, pin, pout, n, code, _OPS[op], int(chunk_bytes),
                                     _stream_handle(stream)), "hvd_allreduce_host")
        return outs

    def allreduce_buffer(self, count: int, dtype: int = HVD_FLOAT32, op: str = "sum", stream=None):
        """Raw ring on the registered fusion buffer (headline measurement)."""
        check(lib.hvd_allreduce_buffer(self._h, int(count), int(dtype), _OPS[op], _stream_handle(stream)),
              "hvd_allreduce_buffer")

    def broadcast(self, tensors, root: int = 0, stream=None):
        arr, n = self._marshal(tensors)
        check(lib.hvd_broadcast(self._h, arr, n, int(root), _stream_handle(stream)), "hvd_broadcast")
        return tensors

    def allgather(self, inputs, outputs, stream=None):
        if self.local_ranks == 1 and not isinstance(inputs, (list, tuple)):
            inputs, outputs = [inputs], [outputs]
        check(lib.hvd_allgather(self._h, _tensor_array(list(inputs)), _tensor_array(list(outputs)),
                                _stream_handle(stream)), "hvd_allgather")
        return outputs

    # ---------------------------------------------------------------- buffers, stats, knobs
    def fusion_buffer(self, local: int = 0, dtype=None, count=None):
        """A torch view of local rank ``local``'s fusion buffer (library-owned memory)."""
        import torch
        ptr = lib.hvd_fusion_buffer(self._h, int(local))
        if not ptr:
            raise HvdError(_lib.HVD_ERR_INVALID, "hvd_fusion_buffer")
        cap = lib.hvd_fusion_capacity(self._h)
        dtype = dtype or torch.float32
        esz = torch.empty((), dtype=dtype).element_size()
        count = cap // esz if count is None else int(count)
        typestr = {torch.float32: "<f4", torch.bfloat16: "<u2", torch.int32: "<i4", torch.int64: "<i8",
                   torch.uint8: "|u1"}[dtype]

        class _View:
            __cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (ptr, False),
                                        "version": 3, "strides": None}
        t = torch.as_tensor(_View(), device=f"cuda:{self.device}")
        return t.view(torch.bfloat16) if dtype == torch.bfloat16 else t

    @property
    def fusion_capacity(self) -> int:
        return lib.hvd_fusion_capacity(self._h)

    def traffic(self, local: int = 0):
        sent, sends = C.c_uint64(), C.c_uint64()
        check(lib.hvd_traffic(self._h, int(local), C.byref(sent), C.byref(sends)), "hvd_traffic")
        return sent.value, sends.value

    def kernel_stats(self):
        """{kind: (launches, device_ms)} since the last call (ms needs HVD_CFG_PROFILE=1)."""
        n = _lib.HVD_KERNEL_KINDS
        la, ms = (C.c_uint64 * n)(), (C.c_double * n)()
        check(lib.hvd_kernel_stats(self._h, la, ms), "hvd_kernel_stats")
        names = ["pack", "ring", "unpack", "scale", "fused", "copy", "pull", "ll", "solo", "ll128", "bulk"]
        return {names[i]: (la[i], ms[i]) for i in range(n)}

    def timeline(self, local: int = 0):
        """Device timeline of the most recent fused launch (needs HVD_CFG_TIMELINE > 0).

        Returns {"rank", "size", "K", "T", "channels", "data": [ch][slice] -> (t0, t1) ns,
        "signals": [ch][j] -> (t, slices_published)} or None if nothing was recorded.
        """
        import numpy as np
        info = _lib.hvd_timeline_info()
        check(lib.hvd_timeline(self._h, int(local), None, 0, C.byref(info)), "hvd_timeline")
        if info.channels == 0:
            return None
        words = _lib.MAX_CHANNELS * info.words_per_channel * 2
        buf = np.zeros(words, dtype=np.uint64)
        check(lib.hvd_timeline(self._h, int(local), buf.ctypes.data_as(C.POINTER(C.c_uint64)), words,
                               C.byref(info)), "hvd_timeline")
        wpc = info.words_per_channel
        data = buf[:_lib.MAX_CHANNELS * wpc].reshape(_lib.MAX_CHANNELS, wpc // 2, 2)[:info.channels, :info.slices]
        sig = buf[_lib.MAX_CHANNELS * wpc:].reshape(_lib.MAX_CHANNELS, wpc // 2, 2)[:info.channels, :info.signals]
        return {"rank": info.rank, "size": info.size, "K": info.K, "T": info.T, "channels": info.channels,
                "kind": {1: "pull", 2: "registered"}.get(info.kind, "push"), "fin_lag": self.get_config(_lib.HVD_CFG_FIN_LAG), "data": data.copy(), "signals": sig.copy()}

    def timeline_start(self, path: str, truncate=None, group=None):
        """Job-wide Horovod Timeline into ``path`` (``hvd_timeline_start``; the environment
        variable ``HVD_TIMELINE=<path>`` does the same at init).  Collective in a
        multi-process job: rank 0 starts a new file (``truncate`` None) and the other
        ranks append after it, ordered by a barrier over ``group``."""
        multi = self.size > 1 and self.local_ranks == 1
        if truncate is None:
            truncate = self.rank == 0
        if multi:
            import torch.distributed as dist
        if not multi or truncate:
            check(lib.hvd_timeline_start(self._h, os.fsencode(path), int(bool(truncate))), "hvd_timeline_start")
        if multi:
            dist.barrier(group)
            if not truncate:
                check(lib.hvd_timeline_start(self._h, os.fsencode(path), 0), "hvd_timeline_start")

    def timeline_stop(self):
        """Synchronise, write every remaining record and close the job timeline."""
        check(lib.hvd_timeline_stop(self._h), "hvd_timeline_stop")

    def timeline_flush(self):
        """Write the records of finished launches; returns (launches traced, records dropped)."""
        la, dr = C.c_uint64(0), C.c_uint64(0)
        check(lib.hvd_timeline_flush(self._h, C.byref(la), C.byref(dr)), "hvd_timeline_flush")
        return la.value, dr.value

    def poll_error(self) -> int:
        return lib.hvd_poll_error(self._h)

    def ll128_selftest(self, force_fail: bool = False) -> int:
        """Collective LL128 line-atomicity self-test (``hvd_ll128_selftest``); returns
        HVD_CFG_LL128_STATUS (1 passed; < 0 failed, LL128 switched off on every rank)."""
        st = C.c_int(0)
        check(lib.hvd_ll128_selftest(self._h, int(bool(force_fail)), C.byref(st)), "hvd_ll128_selftest")
        return st.value

    def set_config(self, key: int, value: int):
        check(lib.hvd_set_config(self._h, int(key), int(value)), "hvd_set_config")

    def get_config(self, key: int) -> int:
        return lib.hvd_get_config(self._h, int(key))

    def finalize(self):
        if self._h:
            lib.hvd_finalize(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.finalize()
        except Exception:
            pass


_DT_NAME = {HVD_FLOAT32: "f32", HVD_BFLOAT16: "bf16", HVD_INT32: "i32", HVD_INT64: "i64"}
_DT_CODE = {v: k for k, v in _DT_NAME.items()}


def plan(counts, dtypes, fusion_threshold=DEFAULT_FUSION_BYTES, capacity=DEFAULT_FUSION_BYTES):
    """The library's Tensor Fusion plan (host-only ``hvd_plan``).

    Returns a list of (dtype, L, [(tensor, src_off, dst_off, count), ...]).
    """
    n = len(counts)
    cc = (C.c_uint64 * max(1, n))(*counts)
    dd = (C.c_int32 * max(1, n))(*[_DT_CODE[d] if isinstance(d, str) else d for d in dtypes])
    ne, nb = C.c_int(0), C.c_int(0)
    lib.hvd_plan(cc, dd, n, int(fusion_threshold), int(capacity), None, C.byref(ne), None, C.byref(nb))
    ents = (_lib.hvd_plan_entry * max(1, ne.value))()
    bufs = (_lib.hvd_plan_buffer * max(1, nb.value))()
    check(lib.hvd_plan(cc, dd, n, int(fusion_threshold), int(capacity), ents, C.byref(ne), bufs, C.byref(nb)),
          "hvd_plan")
    return [(_DT_NAME[b.dtype], b.length,
             [(e.tensor, e.src_off, e.dst_off, e.count) for e in ents[b.first_entry:b.first_entry + b.n_entries]])
            for b in bufs[:nb.value]]


def chunk_bounds(length, size, dtype):
    """The ring's chunk partition of a buffer (host-only ``hvd_chunk_bounds``)."""
    out = (C.c_uint64 * (size + 1))()
    check(lib.hvd_chunk_bounds(int(length), int(size), _DT_CODE[dtype] if isinstance(dtype, str) else dtype, out),
          "hvd_chunk_bounds")
    return list(out)


class Negotiator:
    """Readiness negotiation ("Determine which tensors are ready"; R15):
    ``ready(id)`` as tensors become ready, ``cycle()`` (collective) returns the ids ready on
    every rank, in rank 0's submission order.  Host-only (``hvd_negotiator_*``)."""

    def __init__(self, shm_name, rank: int, size: int, nlocal: int = 1, max_tensors: int = 4096,
                 timeout_ms: int = 60000):
        h = C.c_void_p()
        nm = shm_name.encode() if shm_name else None
        check(lib.hvd_negotiator_create(nm, int(rank), int(size), int(nlocal), int(max_tensors), int(timeout_ms),
                                        C.byref(h)), "hvd_negotiator_create")
        self._h, self.size, self.nlocal, self.max_tensors = h, size, nlocal, max_tensors
        self._ids = (C.c_uint32 * max_tensors)()

    def ready(self, tid: int, count: int, dtype, local: int = 0):
        code = _DT_CODE[dtype] if isinstance(dtype, str) else (dtype if isinstance(dtype, int) else _dtype_code(dtype))
        check(lib.hvd_negotiator_ready(self._h, int(local), int(tid), int(count), code), "hvd_negotiator_ready")

    def ready_tensor(self, tid: int, t, local: int = 0):
        self.ready(tid, t.numel(), _dtype_code(t), local)

    def cycle(self):
        n = C.c_uint32(0)
        check(lib.hvd_negotiator_cycle(self._h, self._ids, C.byref(n)), "hvd_negotiator_cycle")
        return list(self._ids[:n.value])

    def pending(self, local: int = 0):
        n = C.c_uint32(0)
        check(lib.hvd_negotiator_pending(self._h, int(local), self._ids, C.byref(n)), "hvd_negotiator_pending")
        return list(self._ids[:n.value])

    def trace(self, local: int = 0):
        """Negotiation records since the last call: [(id, t_ready_ns, t_agreed_ns)] (Timeline)."""
        n = C.c_uint32(0)
        check(lib.hvd_negotiator_trace(self._h, int(local), None, 0, C.byref(n)), "hvd_negotiator_trace")
        buf = (C.c_uint64 * max(1, 3 * n.value))()
        check(lib.hvd_negotiator_trace(self._h, int(local), buf, n.value, C.byref(n)), "hvd_negotiator_trace")
        return [(int(buf[3 * i]), int(buf[3 * i + 1]), int(buf[3 * i + 2])) for i in range(n.value)]

    def close(self):
        if self._h:
            lib.hvd_negotiator_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def negotiator(comm: "Comm", max_tensors: int = 4096, timeout_ms: int = 60000, group=None) -> Negotiator:
    """A negotiator for ``comm``'s ranks: a process-private one for a virtual comm, else a
    shared-memory segment named by rank 0 and passed over ``group`` (one node)."""
    if comm.local_ranks > 1 or comm.size == 1:
        return Negotiator(None, 0, comm.size, comm.local_ranks, max_tensors, timeout_ms)
    import torch.distributed as dist
    name = [f"/hvd_neg_{os.getpid()}_{os.urandom(4).hex()}" if comm.rank == 0 else None]
    dist.broadcast_object_list(name, src=0, group=group)
    return Negotiator(name[0], comm.rank, comm.size, 1, max_tensors, timeout_ms)


def init_virtual(size: int, device: int = 0, fusion_bytes: int = DEFAULT_FUSION_BYTES) -> Comm:
    """All ``size`` ring ranks simulated on one GPU (same kernels, same signals)."""
    h = C.c_void_p()
    check(lib.hvd_init_virtual(int(size), int(device), int(fusion_bytes), C.byref(h)), "hvd_init_virtual")
    return Comm(h, device)


def exchange_blobs(blob: bytes, group=None):
    """Gather every rank's IPC blob in rank order over a torch.distributed group."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, blob, group=group)
    return out


def init(fusion_bytes: int = DEFAULT_FUSION_BYTES, device: int | None = None, group=None,
         pull_buffers: bool = False) -> Comm:
    """``hvd.init()`` for one process per GPU.

    Reads RANK / WORLD_SIZE / LOCAL_RANK from the environment (torchrun), pins
    the GPU to the local rank, allocates the buffers and maps the
    ring successor through CUDA IPC; blobs travel over ``group`` (a gloo group
    is created if torch.distributed is not initialised).  ``pull_buffers`` also
    allocates the pull protocol's buffers (HVD_CFG_PULL_BUFFERS, needed for
    HVD_CFG_PROTOCOL = 0); every rank must pass the same value.
    """
    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    device = local if device is None else device
    torch.cuda.set_device(device)
    h = C.c_void_p()
    check(lib.hvd_init(rank, world, device, int(fusion_bytes), C.byref(h)), "hvd_init")
    comm = Comm(h, device)
    if pull_buffers:
        comm.set_config(_lib.HVD_CFG_PULL_BUFFERS, 1)
    if world > 1:
        if not dist.is_initialized():
            dist.init_process_group("gloo")
        ln = C.c_uint64(0)
        check(lib.hvd_get_ipc_blob(h, None, C.byref(ln)))
        buf = C.create_string_buffer(ln.value)
        check(lib.hvd_get_ipc_blob(h, buf, C.byref(ln)), "hvd_get_ipc_blob")
        blobs = exchange_blobs(bytes(buf.raw), group)
        joined = b"".join(blobs)
        check(lib.hvd_connect(h, joined, ln.value), "hvd_connect")
        dist.barrier(group)
    return comm

"""ctypes binding of ``libhvd_b200.so`` (include/hvd.h).

Argument marshalling only: no arithmetic of the method lives in Python.  If
the library is missing this module raises at import — there is no fallback.
"""
from __future__ import annotations

import ctypes as C
import pathlib

LIB_PATH = pathlib.Path(__file__).resolve().parent / "libhvd_b200.so"

HVD_OK = 0
HVD_ERR_INVALID = -1
HVD_ERR_UNSUPPORTED = -2
HVD_ERR_CUDA = -3
HVD_ERR_NOT_CONNECTED = -4
HVD_ERR_TIMEOUT = -5
HVD_ERR_CLOSED = -6
HVD_ERR_MISMATCH = -7

HVD_FLOAT32, HVD_BFLOAT16, HVD_INT32, HVD_INT64 = 1, 2, 3, 4
HVD_SUM, HVD_AVERAGE = 0, 1

HVD_CFG_CHANNELS = 1
HVD_CFG_SLICE_BYTES = 2
HVD_CFG_THREADS = 3
HVD_CFG_TIMEOUT_MS = 4
HVD_CFG_PACK_CTAS_PER_SM = 5
HVD_CFG_PROFILE = 6
HVD_CFG_SIGNAL_MODE = 7
HVD_CFG_FUSED = 8
HVD_CFG_TIMELINE = 9
HVD_CFG_WINDOW = 10
HVD_CFG_FIN_LAG = 11
HVD_CFG_PROTOCOL = 12
HVD_CFG_MULTI_BUFFERS = 13
HVD_CFG_LL_MAX_BYTES = 14
HVD_CFG_LL128_MAX_BYTES = 15
HVD_CFG_BULK_STAGES = 16
HVD_CFG_BULK_STAGE_BYTES = 17
HVD_CFG_BULK_DEPTH = 18
HVD_CFG_BULK_CHANNELS = 19
HVD_CFG_BULK_SLICE_BYTES = 20
HVD_CFG_SIGNAL_WARPS = 21
HVD_CFG_LL128_STATUS = 22
HVD_CFG_SOLO_KERNEL = 23
HVD_CFG_SOLO_STAGES = 24
HVD_CFG_SOLO_STAGE_BYTES = 25
HVD_CFG_PACE_GBPS = 26
HVD_CFG_PACE_BURST_ROWS = 27
HVD_CFG_FUSED_PDL = 28
HVD_CFG_WATCHER = 29
HVD_CFG_HOST_ZERO_COPY = 30
HVD_CFG_PREISSUE = 31
HVD_CFG_LL_PDL = 32
HVD_CFG_PULL_BUFFERS = 33
HVD_CFG_SOLO_TAIL = 34
MAX_CHANNELS = 256
HVD_KERNEL_PACK, HVD_KERNEL_RING, HVD_KERNEL_UNPACK, HVD_KERNEL_SCALE, HVD_KERNEL_FUSED = 0, 1, 2, 3, 4
HVD_KERNEL_COPY = 5
HVD_KERNEL_PULL = 6
HVD_KERNEL_LL = 7
HVD_KERNEL_SOLO = 8
HVD_KERNEL_LL128 = 9
HVD_KERNEL_BULK = 10
HVD_KERNEL_KINDS = 11


class hvd_tensor(C.Structure):
    _fields_ = [("data", C.c_void_p), ("count", C.c_uint64), ("dtype", C.c_int32), ("reserved", C.c_int32)]


class hvd_plan_entry(C.Structure):
    _fields_ = [("tensor", C.c_int32), ("buffer", C.c_int32), ("src_off", C.c_uint64),
                ("dst_off", C.c_uint64), ("count", C.c_uint64)]


class hvd_plan_buffer(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("n_entries", C.c_int32), ("first_entry", C.c_int32),
                ("reserved", C.c_int32), ("length", C.c_uint64)]


class hvd_timeline_info(C.Structure):
    _fields_ = [("channels", C.c_int32), ("slices", C.c_int32), ("signals", C.c_int32), ("K", C.c_int32),
                ("T", C.c_int32), ("rank", C.c_int32), ("size", C.c_int32), ("kind", C.c_int32),
                ("words_per_channel", C.c_uint64)]


class HvdError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        super().__init__(f"{what}: {strerror(status)} ({status})" if what else f"{strerror(status)} ({status})")


def _load():
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() "
                          "(python -m paper_1802_05799_b200._build)")
    lib = C.CDLL(str(LIB_PATH))
    P = C.c_void_p
    sig = {
        "hvd_init": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_uint64, C.POINTER(P)]),
        "hvd_init_virtual": (C.c_int, [C.c_int, C.c_int, C.c_uint64, C.POINTER(P)]),
        "hvd_get_ipc_blob": (C.c_int, [P, P, C.POINTER(C.c_uint64)]),
        "hvd_connect": (C.c_int, [P, P, C.c_uint64]),
        "hvd_finalize": (C.c_int, [P]),
        "hvd_rank": (C.c_int, [P]),
        "hvd_size": (C.c_int, [P]),
        "hvd_local_ranks": (C.c_int, [P]),
        "hvd_allreduce": (C.c_int, [P, C.POINTER(hvd_tensor), C.c_int, C.c_int, C.c_uint64, P]),
        "hvd_allreduce_average": (C.c_int, [P, C.POINTER(hvd_tensor), C.c_int, C.c_uint64, P]),
        "hvd_allreduce_ex": (C.c_int, [P, C.POINTER(hvd_tensor), C.c_int, C.c_int, C.c_uint64, C.c_int, P]),
        "hvd_register_blob": (C.c_int, [P, C.POINTER(hvd_tensor), C.c_int, P, C.POINTER(C.c_uint64)]),
        "hvd_register": (C.c_int, [P, C.POINTER(hvd_tensor), C.c_int, P, C.c_uint64, C.POINTER(C.c_int)]),
        "hvd_allreduce_registered": (C.c_int, [P, C.c_int, C.c_int, C.c_uint64, P]),
        "hvd_deregister": (C.c_int, [P, C.c_int]),
        "hvd_allreduce_buffer": (C.c_int, [P, C.c_uint64, C.c_int, C.c_int, P]),
        "hvd_fusion_buffer": (P, [P, C.c_int]),
        "hvd_fusion_capacity": (C.c_uint64, [P]),
        "hvd_broadcast": (C.c_int, [P, C.POINTER(hvd_tensor), C.c_int, C.c_int, P]),
        "hvd_allgather": (C.c_int, [P, C.POINTER(hvd_tensor), C.POINTER(hvd_tensor), P]),
        "hvd_poll_error": (C.c_int, [P]),
        "hvd_strerror": (C.c_char_p, [C.c_int]),
        "hvd_build_id": (C.c_char_p, []),
        "hvd_timeline_start": (C.c_int, [P, C.c_char_p, C.c_int]),
        "hvd_timeline_stop": (C.c_int, [P]),
        "hvd_timeline_flush": (C.c_int, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
        "hvd_traffic": (C.c_int, [P, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
        "hvd_set_config": (C.c_int, [P, C.c_int, C.c_int64]),
        "hvd_get_config": (C.c_int64, [P, C.c_int]),
        "hvd_plan": (C.c_int, [C.POINTER(C.c_uint64), C.POINTER(C.c_int32), C.c_int, C.c_uint64, C.c_uint64,
                               C.POINTER(hvd_plan_entry), C.POINTER(C.c_int), C.POINTER(hvd_plan_buffer),
                               C.POINTER(C.c_int)]),
        "hvd_chunk_bounds": (C.c_int, [C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_uint64)]),
        "hvd_kernel_stats": (C.c_int, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_double)]),
        "hvd_timeline": (C.c_int, [P, C.c_int, C.POINTER(C.c_uint64), C.c_uint64, C.POINTER(hvd_timeline_info)]),
        "hvd_allreduce_host": (C.c_int, [P, C.POINTER(P), C.POINTER(P), C.c_uint64, C.c_int, C.c_int, C.c_uint64,
                                         P]),
        "hvd_negotiator_create": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_uint32, C.c_uint64,
                                            C.POINTER(P)]),
        "hvd_negotiator_ready": (C.c_int, [P, C.c_int, C.c_uint32, C.c_uint64, C.c_int]),
        "hvd_negotiator_cycle": (C.c_int, [P, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
        "hvd_negotiator_pending": (C.c_int, [P, C.c_int, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
        "hvd_negotiator_destroy": (C.c_int, [P]),
        "hvd_negotiator_trace": (C.c_int, [P, C.c_int, C.POINTER(C.c_uint64), C.c_uint32, C.POINTER(C.c_uint32)]),
        "hvd_ll128_selftest": (C.c_int, [P, C.c_int, C.POINTER(C.c_int)]),
        "hvd_allreduce_negotiated": (C.c_int, [P, P, C.POINTER(hvd_tensor), C.c_uint32, C.c_int, C.c_uint64, P,
                                               C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()

# every function declared in include/hvd.h (tests check the export table against this)
EXPORTS = sorted([
    "hvd_init", "hvd_init_virtual", "hvd_get_ipc_blob", "hvd_connect", "hvd_finalize", "hvd_rank",
    "hvd_size", "hvd_local_ranks", "hvd_allreduce", "hvd_allreduce_average", "hvd_allreduce_buffer",
    "hvd_fusion_buffer", "hvd_fusion_capacity", "hvd_broadcast", "hvd_allgather", "hvd_poll_error",
    "hvd_strerror", "hvd_traffic", "hvd_set_config", "hvd_get_config", "hvd_plan", "hvd_chunk_bounds",
    "hvd_kernel_stats", "hvd_timeline", "hvd_allreduce_ex", "hvd_register_blob", "hvd_register",
    "hvd_allreduce_registered", "hvd_deregister", "hvd_negotiator_create", "hvd_negotiator_ready",
    "hvd_negotiator_cycle", "hvd_negotiator_pending", "hvd_negotiator_destroy", "hvd_allreduce_negotiated",
    "hvd_allreduce_host", "hvd_negotiator_trace", "hvd_ll128_selftest", "hvd_build_id",
    "hvd_timeline_start", "hvd_timeline_stop", "hvd_timeline_flush",
])


def strerror(status: int) -> str:
    return lib.hvd_strerror(int(status)).decode()


def check(status: int, what: str = "") -> int:
    if status != HVD_OK:
        raise HvdError(status, what)
    return status

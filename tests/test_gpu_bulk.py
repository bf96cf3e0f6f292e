"""GPU parity of the bulk-copy push ring (``bulk_allreduce_kernel``, HVD_CFG_PROTOCOL=2).

Same virtual-rank setup as ``test_gpu_virtual.py``: all N ranks in one launch on
one B200, every result compared element by element with the CPU oracle
(bit-exact: the kernel reproduces the ring's chunks and reduction order).  The
LL / LL128 latency protocols are switched off where a case must run on the
bulk kernel, and the launch counters prove which kernel ran.
"""
import numpy as np
import pytest

import oracle
import workloads
from hvd_testutil import HVD_CODE, assert_same, from_torch, to_torch

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def hvd():
    import paper_1802_05799_b200 as m
    return m


_COMMS = {}


@pytest.fixture(scope="module", autouse=True)
def _finalize_comms():
    """Each virtual comm holds every rank's buffers on the one GPU: free them per module."""
    yield
    for c in _COMMS.values():
        c.finalize()
    _COMMS.clear()


def bulk_comm(hvd, n, cap=64 << 20, ll=False, proto=2):
    key = (n, cap, ll, proto)
    if key not in _COMMS:
        c = hvd.init_virtual(n, 0, cap)
        L = hvd._lib
        c.set_config(L.HVD_CFG_TIMEOUT_MS, 20000)
        c.set_config(L.HVD_CFG_PROTOCOL, proto)
        if not ll:
            c.set_config(L.HVD_CFG_LL_MAX_BYTES, 0)
            c.set_config(L.HVD_CFG_LL128_MAX_BYTES, 0)
        _COMMS[key] = c
    return _COMMS[key]


def _tensors(xs, dtypes, misalign_rank=None):
    keep, ts = [], []
    for r, row in enumerate(xs):
        out = []
        for x, dt in zip(row, dtypes):
            t = to_torch(x, dt)
            if misalign_rank is not None and r == misalign_rank and len(x) > 0:
                big = torch.empty(len(x) + 1, dtype=t.dtype, device="cuda")
                big[1:].copy_(t)
                keep.append(big)
                t = big[1:]
            out.append(t)
        ts.append(out)
    return ts, keep


RAGGED = [1, 3, 64, 1000, 4097, 100_003, 7, 262_149, 0, 33]


@pytest.mark.parametrize("n", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_bulk_average_ragged_multibuffer(hvd, n, dtype):
    """Ragged member ends (element-wise pieces) and several fusion buffers per launch."""
    comm = bulk_comm(hvd, n)
    xs = workloads.all_ranks(RAGGED, dtype, n)
    dts = [dtype] * len(RAGGED)
    ref, _, plan = oracle.allreduce(xs, dts, "average", threshold=400_000)
    assert len(plan) > 1
    ts, _ = _tensors(xs, dts)
    comm.kernel_stats()
    comm.allreduce(ts, op="average", fusion_threshold=400_000)
    torch.cuda.synchronize()
    assert comm.poll_error() == 0
    st = comm.kernel_stats()
    assert st["bulk"][0] >= 1 and st["fused"][0] == 0
    for r in range(n):
        for k in range(len(RAGGED)):
            assert_same(from_torch(ts[r][k], dtype), ref[r][k], dtype, f"N={n} r={r} k={k}")


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("dtype", ["i32", "i64"])
def test_bulk_integer_sum_exact(hvd, n, dtype):
    comm = bulk_comm(hvd, n)
    xs = workloads.all_ranks(RAGGED, dtype, n, kind="int_uniform")
    dts = [dtype] * len(RAGGED)
    ref, _, _ = oracle.allreduce(xs, dts, "sum")
    ts, _ = _tensors(xs, dts)
    comm.allreduce(ts, op="sum")
    torch.cuda.synchronize()
    assert comm.poll_error() == 0
    for r in range(n):
        for k in range(len(RAGGED)):
            assert_same(from_torch(ts[r][k], dtype), ref[r][k], dtype, f"N={n} r={r} k={k}")


@pytest.mark.parametrize("n", [2, 4])
def test_bulk_misaligned_tensors_one_rank(hvd, n):
    """A tensor view off the 16 B grid on one rank: its pieces go element by element there."""
    comm = bulk_comm(hvd, n)
    counts = [5, 17, 1024, 3, 65_537, 300_000]
    xs = workloads.all_ranks(counts, "f32", n)
    dts = ["f32"] * len(counts)
    ref, _, _ = oracle.allreduce(xs, dts, "average")
    ts, keep = _tensors(xs, dts, misalign_rank=n - 1)
    comm.allreduce(ts, op="average")
    torch.cuda.synchronize()
    assert comm.poll_error() == 0
    for r in range(n):
        for k in range(len(counts)):
            assert_same(from_torch(ts[r][k], "f32"), ref[r][k], "f32", f"r={r} k={k}")


@pytest.mark.parametrize("stages,stage_kib,depth,slice_kib,channels",
                         [(3, 4, 0, 4, 7), (4, 8, 1, 16, 33), (6, 16, 3, 64, 148), (3, 32, 1, 256, 64),
                          (5, 4, 2, 1, 148)])
def test_bulk_geometry_knobs_keep_bits(hvd, stages, stage_kib, depth, slice_kib, channels):
    """Stage size / count / depth, slice and channel count change the schedule, never the bits.
    4 KiB stages with many small members also exercise the stage cut at a full exception list."""
    n = 3
    comm = hvd.init_virtual(n, 0, 8 << 20)
    try:
        L = hvd._lib
        for k, v in ((L.HVD_CFG_TIMEOUT_MS, 20000), (L.HVD_CFG_PROTOCOL, 2), (L.HVD_CFG_LL_MAX_BYTES, 0),
                     (L.HVD_CFG_LL128_MAX_BYTES, 0), (L.HVD_CFG_BULK_DEPTH, 0), (L.HVD_CFG_BULK_STAGES, stages),
                     (L.HVD_CFG_BULK_DEPTH, depth), (L.HVD_CFG_BULK_STAGE_BYTES, stage_kib << 10),
                     (L.HVD_CFG_BULK_SLICE_BYTES, slice_kib << 10), (L.HVD_CFG_BULK_CHANNELS, channels)):
            comm.set_config(k, v)
        counts = [1_000_003, 4096] + [int(c) for c in np.random.default_rng(3).integers(1, 50, size=300)]
        xs = workloads.all_ranks(counts, "f32", n)
        ref, _, _ = oracle.allreduce(xs, ["f32"] * len(counts), "average")
        ts, _ = _tensors(xs, ["f32"] * len(counts))
        comm.kernel_stats()
        comm.allreduce_average(ts)
        torch.cuda.synchronize()
        assert comm.poll_error() == 0
        assert comm.kernel_stats()["bulk"][0] == 1
        for r in range(n):
            for k in range(len(counts)):
                assert_same(from_torch(ts[r][k], "f32"), ref[r][k], "f32", f"cfg r={r} k={k}")
    finally:
        comm.finalize()


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_bulk_registered_zero_copy(hvd, n):
    """Registered tensors: the all-gather bulk-stores final values into the successor's tensors."""
    comm = hvd.init_virtual(n, 0, 1 << 20)
    try:
        L = hvd._lib
        for k, v in ((L.HVD_CFG_TIMEOUT_MS, 20000), (L.HVD_CFG_PROTOCOL, 2), (L.HVD_CFG_LL_MAX_BYTES, 0),
                     (L.HVD_CFG_LL128_MAX_BYTES, 0)):
            comm.set_config(k, v)
        counts = [3, 1000, 262_149, 5, 77_777, 400_001]
        ts = [[torch.empty(c, device="cuda") for c in counts] for _ in range(n)]
        keep = [torch.empty(1001, device="cuda")]
        ts[0][1] = keep[0][1:]  # a misaligned view on one rank
        reg = comm.register(ts)
        for it in range(3):
            xs = workloads.all_ranks(counts, "f32", n, seed=900 + it)
            for r in range(n):
                for k in range(len(counts)):
                    ts[r][k].copy_(to_torch(xs[r][k], "f32"))
            ref, _, _ = oracle.allreduce(xs, ["f32"] * len(counts), "average", threshold=1 << 19, capacity=1 << 20)
            comm.kernel_stats()
            comm.allreduce_average(reg, fusion_threshold=1 << 19)
            torch.cuda.synchronize()
            assert comm.poll_error() == 0
            assert comm.kernel_stats()["bulk"][0] >= 1
            for r in range(n):
                for k in range(len(counts)):
                    assert_same(from_torch(ts[r][k], "f32"), ref[r][k], "f32", f"it={it} r={r} k={k}")
        comm.deregister(reg)
    finally:
        comm.finalize()


KERNEL = {1: "fused", 2: "bulk"}


@pytest.mark.parametrize("proto", [1, 2])
@pytest.mark.parametrize("n", [2, 4, 8])
def test_bench_step_registered_64MiB(hvd, n, proto):
    """bench.py's exact step: one registered 64 MiB fp32 gradient, default 64 MiB capacity,
    allreduce-average through the default SM-store push (1) and the bulk push (2); every
    element vs the oracle."""
    comm = bulk_comm(hvd, n, ll=True, proto=proto)
    cnt = 16 << 20
    xs = [[workloads.rank_tensor(cnt, "f32", r, 0)] for r in range(n)]
    ref, _, plan = oracle.allreduce(xs, ["f32"], "average")
    assert len(plan) == 1
    ts = [[to_torch(xs[r][0], "f32")] for r in range(n)]
    reg = comm.register(ts)
    comm.kernel_stats()
    comm.allreduce_average(reg)
    torch.cuda.synchronize()
    assert comm.poll_error() == 0
    assert comm.kernel_stats()[KERNEL[proto]][0] == 1
    for r in range(n):
        assert_same(from_torch(ts[r][0], "f32"), ref[r][0], "f32", f"N={n} r={r}")
    comm.deregister(reg)


@pytest.mark.parametrize("proto", [1, 2])
@pytest.mark.parametrize("n", [2, 4, 8])
def test_raw_buffer_16Mi_and_traffic(hvd, n, proto):
    """hvd_allreduce_buffer of 16 Mi fp32 (the headline ring) and a ragged length: bits and the
    per-rank traffic counters 2L - |c_{r+1}| - |c_{r+2}|."""
    comm = bulk_comm(hvd, n, proto=proto)
    for L_ in (16 << 20, 3_000_017):
        xs = [workloads.rank_tensor(L_, "f32", r, 9) for r in range(n)]
        ref, tr = oracle.allreduce_buffer(xs, "f32", "average")
        before = [comm.traffic(r) for r in range(n)]
        for r in range(n):
            comm.fusion_buffer(r, torch.float32, L_).copy_(to_torch(xs[r], "f32"))
        comm.allreduce_buffer(L_, HVD_CODE["f32"], "average")
        torch.cuda.synchronize()
        assert comm.poll_error() == 0
        for r in range(n):
            assert_same(from_torch(comm.fusion_buffer(r, torch.float32, L_), "f32"), ref[r], "f32", f"L={L_} r={r}")
            sent, sends = comm.traffic(r)
            assert sent - before[r][0] == tr[r].sent_elems * 4
            assert sends - before[r][1] == 2 * (n - 1)


@pytest.mark.parametrize("proto", [1, 2])
@pytest.mark.parametrize("model,dtype,n", [("vgg16", "f32", 4), ("vgg16", "f32", 8), ("resnet101", "f32", 4),
                                           ("inception_v3", "bf16", 2)])
def test_model_sets_full_size(hvd, model, dtype, n, proto):
    """BASELINE configs C2-C4 at full size (VGG-16: 11 buffers, fc6 split 6 x 64 + 8 MiB, fc7
    exactly 64 MiB), library defaults (LL / LL128 for small buffers) with the SM-store push (1)
    or the bulk push (2) for the rest: every element vs the oracle."""
    comm = bulk_comm(hvd, n, ll=True, proto=proto)
    counts = [c for _, c in workloads.gradient_set(model)]
    xs = workloads.all_ranks(counts, dtype, n)
    dts = [dtype] * len(counts)
    ref, _, plan = oracle.allreduce(xs, dts, "average")
    if model == "vgg16":
        assert len(plan) == 11
    ts, _ = _tensors(xs, dts)
    comm.allreduce(ts, op="average")
    torch.cuda.synchronize()
    assert comm.poll_error() == 0
    for r in range(n):
        for k in range(len(counts)):
            assert_same(from_torch(ts[r][k], dtype), ref[r][k], dtype, f"{model} r={r} k={k}")


def test_bulk_back_to_back_mixed_protocols(hvd):
    """Bulk, fused, LL and LL128 launches back to back without host syncs: counters and receive
    regions hand over between kernels."""
    n = 4
    comm = hvd.init_virtual(n, 0, 64 << 20)
    try:
        L = hvd._lib
        comm.set_config(L.HVD_CFG_TIMEOUT_MS, 20000)
        pend = []
        for i, (proto, counts) in enumerate([(2, [5_000_000]), (1, [3_000_000, 17]), (2, [100, 70_000]),
                                             (2, [9_000_001]), (1, [1 << 20]), (2, [12_345_679, 8])]):
            comm.set_config(L.HVD_CFG_PROTOCOL, proto)
            xs = workloads.all_ranks(counts, "f32", n, seed=2000 + i)
            ts, _ = _tensors(xs, ["f32"] * len(counts))
            comm.allreduce_average(ts)
            pend.append((xs, ts))
        torch.cuda.synchronize()
        assert comm.poll_error() == 0
        for xs, ts in pend:
            ref, _, _ = oracle.allreduce(xs, ["f32"] * len(xs[0]), "average")
            for r in range(n):
                for k in range(len(xs[0])):
                    assert_same(from_torch(ts[r][k], "f32"), ref[r][k], "f32")
    finally:
        comm.finalize()

"""GPU parity of the fused ring allreduce with N ranks simulated on one B200.

``hvd_init_virtual`` runs the SAME kernels and signal protocol as the
multi-process path (one launch spans every rank, so the ranks' CTAs are
co-resident); "peer" buffers are same-device allocations.  Every result is
compared element by element with the CPU oracle on the same seeded inputs
(bit-exact: the ring order is reproduced).
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


def comm_for(hvd, n, cap=64 << 20):
    key = (n, cap)
    if key not in _COMMS:
        c = hvd.init_virtual(n, 0, cap)
        c.set_config(hvd._lib.HVD_CFG_TIMEOUT_MS, 20000)
        _COMMS[key] = c
    return _COMMS[key]


def run_allreduce(hvd, xs, dtypes, op, threshold, cap=64 << 20, misalign=False):
    n = len(xs)
    comm = comm_for(hvd, n, cap)
    ts = []
    keep = []
    for r in range(n):
        row = []
        for x, dt in zip(xs[r], dtypes):
            t = to_torch(x, dt)
            if misalign and len(x) > 0:      # a view whose data_ptr is off the 16 B grid
                big = torch.empty(len(x) + 1, dtype=t.dtype, device="cuda")
                big[1:].copy_(t)
                keep.append(big)
                t = big[1:]
            row.append(t)
        ts.append(row)
    comm.allreduce(ts, op=op, fusion_threshold=threshold)
    torch.cuda.synchronize()
    assert comm.poll_error() == 0
    return [[from_torch(t, dt) for t, dt in zip(ts[r], dtypes)] for r in range(n)]


RAGGED = [1, 3, 64, 1000, 4097, 100_003, 7, 262_149, 0, 33]


@pytest.mark.parametrize("n", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_allreduce_average_bitexact(hvd, n, dtype):
    xs = workloads.all_ranks(RAGGED, dtype, n)
    dts = [dtype] * len(RAGGED)
    ref, _, plan = oracle.allreduce(xs, dts, "average", threshold=400_000)
    assert len(plan) > 1
    got = run_allreduce(hvd, xs, dts, "average", 400_000)
    for r in range(n):
        for k in range(len(RAGGED)):
            assert_same(got[r][k], ref[r][k], dtype, f"N={n} r={r} k={k}")


@pytest.mark.parametrize("n", [2, 3, 4, 8])
@pytest.mark.parametrize("dtype", ["i32", "i64"])
def test_allreduce_sum_integers_exact(hvd, n, dtype):
    xs = workloads.all_ranks(RAGGED, dtype, n, kind="int_uniform")
    dts = [dtype] * len(RAGGED)
    ref, _, _ = oracle.allreduce(xs, dts, "sum")
    got = run_allreduce(hvd, xs, dts, "sum", 64 << 20)
    for r in range(n):
        for k in range(len(RAGGED)):
            assert_same(got[r][k], ref[r][k], dtype, f"N={n} r={r} k={k}")


@pytest.mark.parametrize("n", [1, 2, 4])
def test_fusion_off_and_misaligned_tensors(hvd, n):
    counts = [5, 17, 1024, 3, 65_537]
    xs = workloads.all_ranks(counts, "f32", n)
    dts = ["f32"] * len(counts)
    ref, _, plan = oracle.allreduce(xs, dts, "average", threshold=0)
    assert len(plan) == len(counts)
    got = run_allreduce(hvd, xs, dts, "average", 0, misalign=True)
    for r in range(n):
        for k in range(len(counts)):
            assert_same(got[r][k], ref[r][k], "f32", f"r={r} k={k}")


@pytest.mark.parametrize("n", [2, 3, 8])
def test_mixed_dtype_list(hvd, n):
    counts = [100, 200, 300, 400, 5000]
    dts = ["f32", "bf16", "f32", "bf16", "bf16"]
    xs = [[workloads.rank_tensor(c, d, r, k) for k, (c, d) in enumerate(zip(counts, dts))] for r in range(n)]
    ref, _, _ = oracle.allreduce(xs, dts, "average")
    got = run_allreduce(hvd, xs, dts, "average", 64 << 20)
    for r in range(n):
        for k in range(len(counts)):
            assert_same(got[r][k], ref[r][k], dts[k], f"r={r} k={k}")


@pytest.mark.parametrize("n", [2, 4])
def test_specials_and_rank_agreement(hvd, n):
    counts = [5000, 77]
    for dt in ("f32", "bf16"):
        xs = workloads.all_ranks(counts, dt, n, kind="specials")
        ref, _, _ = oracle.allreduce(xs, [dt, dt], "average")
        got = run_allreduce(hvd, xs, [dt, dt], "average", 64 << 20)
        for r in range(n):
            for k in range(2):
                assert_same(got[r][k], ref[r][k], dt, f"{dt} r={r} k={k}")
                assert np.array_equal(got[r][k].view(np.uint8), got[0][k].view(np.uint8))


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_raw_buffer_ring_and_traffic(hvd, n):
    comm = comm_for(hvd, n)
    for dtype in ("f32", "bf16", "i32", "i64"):
        esz = oracle.ELEM_SIZE[dtype]
        for L in (1, 64 * n - 1, 1 << 16, 3_000_017 // esz):
            kind = "normal" if dtype in ("f32", "bf16") else "int_uniform"
            xs = [workloads.rank_tensor(L, dtype, r, 9, kind) for r in range(n)]
            op = "average" if dtype in ("f32", "bf16") else "sum"
            ref, tr = oracle.allreduce_buffer(xs, dtype, op)
            before = [comm.traffic(r) for r in range(n)]
            tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "i32": torch.int32, "i64": torch.int64}[dtype]
            for r in range(n):
                comm.fusion_buffer(r, tdt, L).copy_(to_torch(xs[r], dtype))
            comm.allreduce_buffer(L, HVD_CODE[dtype], op)
            torch.cuda.synchronize()
            for r in range(n):
                got = from_torch(comm.fusion_buffer(r, tdt, L), dtype)
                assert_same(got, ref[r], dtype, f"{dtype} L={L} r={r}")
                sent, sends = comm.traffic(r)
                assert sent - before[r][0] == tr[r].sent_elems * esz
                assert sends - before[r][1] == tr[r].sends == 2 * (n - 1)


def test_back_to_back_calls_varying_sizes(hvd):
    """Monotone signal epochs: consecutive calls of different shapes, no resets."""
    n = 4
    comm = comm_for(hvd, n)
    sizes = [[10], [1 << 20, 5], [3], [70_000, 70_001, 9], [1 << 22]]
    pend = []
    for i, counts in enumerate(sizes):
        xs = workloads.all_ranks(counts, "f32", n, seed=1000 + i)
        ts = [[to_torch(x, "f32") for x in xs[r]] for r in range(n)]
        comm.allreduce_average(ts)
        pend.append((xs, ts))
    torch.cuda.synchronize()
    assert comm.poll_error() == 0
    for xs, ts in pend:
        ref, _, _ = oracle.allreduce(xs, ["f32"] * len(xs[0]), "average")
        for r in range(n):
            for k in range(len(xs[0])):
                assert_same(from_torch(ts[r][k], "f32"), ref[r][k], "f32")


def test_tuning_knobs_keep_bits(hvd):
    """Channels / slice / threads change the schedule of work, never the result."""
    n = 3
    comm = hvd.init_virtual(n, 0, 8 << 20)
    try:
        counts = [1_000_003, 4096]
        xs = workloads.all_ranks(counts, "f32", n)
        ref, _, _ = oracle.allreduce(xs, ["f32", "f32"], "average")
        L = hvd._lib
        comm.set_config(L.HVD_CFG_LL_MAX_BYTES, 0)  # one small buffer: keep it on the fused kernel
        comm.set_config(L.HVD_CFG_LL128_MAX_BYTES, 0)
        for ch, sl, th in [(1, 256, 64), (7, 4096, 256), (64, 1 << 20, 384), (16, 65536, 128), (256, 512, 96)]:
            comm.set_config(L.HVD_CFG_CHANNELS, ch)
            comm.set_config(L.HVD_CFG_SLICE_BYTES, sl)
            comm.set_config(L.HVD_CFG_THREADS, th)
            ts = [[to_torch(x, "f32") for x in xs[r]] for r in range(n)]
            comm.allreduce_average(ts)
            torch.cuda.synchronize()
            for r in range(n):
                for k in range(2):
                    assert_same(from_torch(ts[r][k], "f32"), ref[r][k], "f32", f"cfg {ch},{sl},{th}")
        # remote-store pacing, programmatic dependent launch: timing knobs, same bits
        comm.set_config(L.HVD_CFG_CHANNELS, 32)
        comm.set_config(L.HVD_CFG_SLICE_BYTES, 0)
        comm.set_config(L.HVD_CFG_THREADS, 256)
        for key, val in ((L.HVD_CFG_PACE_GBPS, 300), (L.HVD_CFG_PACE_BURST_ROWS, 0), (L.HVD_CFG_FUSED_PDL, 1),
                         (L.HVD_CFG_WATCHER, 1), (L.HVD_CFG_PREISSUE, 1), (L.HVD_CFG_WATCHER, 0),
                         (L.HVD_CFG_LL_PDL, 1)):
            comm.set_config(key, val)
            for _ in range(2):  # back to back (PDL overlaps the launches)
                ts = [[to_torch(x, "f32") for x in xs[r]] for r in range(n)]
                comm.allreduce_average(ts)
            torch.cuda.synchronize()
            assert comm.poll_error() == 0
            for r in range(n):
                for k in range(2):
                    assert_same(from_torch(ts[r][k], "f32"), ref[r][k], "f32", f"knob {key}={val}")
    finally:
        comm.finalize()


@pytest.mark.parametrize("n", [2, 4])
def test_ll_pdl_back_to_back(hvd, n):
    """HVD_CFG_LL_PDL: LL and LL128 launches back to back without host syncs, each launch
    scheduled while the previous one drains; same bits as the oracle."""
    comm = comm_for(hvd, n)
    L = hvd._lib
    comm.set_config(L.HVD_CFG_LL_PDL, 1)  # (the default)
    try:
        cases = [[1000, 3001], [300_001], [7], [1_000_003], [65_536, 5]]
        runs = []
        for it in range(2):
            for k, counts in enumerate(cases):
                xs = workloads.all_ranks(counts, "f32", n, seed=500 + 10 * it + k)
                ts = [[to_torch(x, "f32") for x in xs[r]] for r in range(n)]
                comm.allreduce(ts, op="average")
                runs.append((xs, ts, counts))
        torch.cuda.synchronize()
        assert comm.poll_error() == 0
        st = comm.kernel_stats()
        assert st["ll"][0] >= 1 and st["ll128"][0] >= 1
        for xs, ts, counts in runs:
            ref, _, _ = oracle.allreduce(xs, ["f32"] * len(counts), "average")
            for r in range(n):
                for k in range(len(counts)):
                    assert_same(from_torch(ts[r][k], "f32"), ref[r][k], "f32", f"{counts} r={r} k={k}")
    finally:
        comm.set_config(L.HVD_CFG_LL_PDL, 1)


def test_errors_on_device(hvd):
    comm = comm_for(hvd, 2)
    t = [[torch.zeros(4, dtype=torch.int32, device="cuda")] for _ in range(2)]
    with pytest.raises(hvd.HvdError) as e:
        comm.allreduce(t, op="average")
    assert e.value.status == hvd._lib.HVD_ERR_UNSUPPORTED
    bad = [[torch.zeros(4, device="cuda")], [torch.zeros(5, device="cuda")]]
    with pytest.raises(hvd.HvdError):
        comm.allreduce(bad, op="sum")
    with pytest.raises(hvd.HvdError):
        comm.allreduce_buffer(comm.fusion_capacity // 4 + 1)
    comm.allreduce([[], []])  # n = 0 is a no-op
    assert comm.poll_error() == 0


@pytest.mark.parametrize("model,dtype,n", [("resnet101", "f32", 4), ("inception_v3", "bf16", 2),
                                           ("inception_v3", "f32", 8)])
def test_model_gradient_sets_full_size(hvd, model, dtype, n):
    """BASELINE configs at full size: every element vs the oracle."""
    counts = [c for _, c in workloads.gradient_set(model)]
    xs = workloads.all_ranks(counts, dtype, n)
    dts = [dtype] * len(counts)
    ref, _, plan = oracle.allreduce(xs, dts, "average")
    got = run_allreduce(hvd, xs, dts, "average", 64 << 20)
    for r in range(n):
        for k in range(len(counts)):
            assert_same(got[r][k], ref[r][k], dtype, f"{model} r={r} k={k}")


@pytest.mark.parametrize("n", [1, 2, 3, 8])
def test_three_kernel_path_bitexact(hvd, n):
    """HVD_CFG_FUSED=0: pack -> ring -> unpack as three launches; same bits as the fused kernel."""
    comm = hvd.init_virtual(n, 0, 4 << 20)
    try:
        comm.set_config(hvd._lib.HVD_CFG_FUSED, 0)
        counts = [3, 1000, 262_149, 5, 77_777]
        xs = workloads.all_ranks(counts, "f32", n)
        ref, _, plan = oracle.allreduce(xs, ["f32"] * len(counts), "average", threshold=1 << 20, capacity=4 << 20)
        ts = [[to_torch(x, "f32") for x in xs[r]] for r in range(n)]
        comm.allreduce(ts, op="average", fusion_threshold=1 << 20)
        torch.cuda.synchronize()
        st = comm.kernel_stats()
        assert st["fused"][0] == 0 and st["pack"][0] == len(plan) and st["unpack"][0] == len(plan)
        for r in range(n):
            for k in range(len(counts)):
                assert_same(from_torch(ts[r][k], "f32"), ref[r][k], "f32", f"r={r} k={k}")
    finally:
        comm.finalize()


@pytest.mark.parametrize("n", [2, 4])
def test_large_plan_global_segment_table(hvd, n):
    """> 4096 members per fusion buffer: the fused kernel reads the member table from global memory."""
    counts = [int(c) for c in np.random.default_rng(5).integers(1, 40, size=5000)]
    xs = workloads.all_ranks(counts, "bf16", n)
    ref, _, plan = oracle.allreduce(xs, ["bf16"] * len(counts), "average")
    assert len(plan) == 1 and len(plan[0].entries) > 4096
    got = run_allreduce(hvd, xs, ["bf16"] * len(counts), "average", 64 << 20)
    for r in range(n):
        for k in range(0, len(counts), 7):
            assert_same(got[r][k], ref[r][k], "bf16", f"r={r} k={k}")


def test_timeline_records_every_slice(hvd):
    """Horovod Timeline: one record per slice op, ordered, plus signals."""
    from paper_1802_05799_b200 import timeline
    n = 3
    comm = hvd.init_virtual(n, 0, 8 << 20)
    try:
        comm.set_config(hvd._lib.HVD_CFG_TIMELINE, 256)
        comm.set_config(hvd._lib.HVD_CFG_PROTOCOL, 1)  # push kernel records
        comm.set_config(hvd._lib.HVD_CFG_LL_MAX_BYTES, 0)  # the LL kernels record no timeline
        comm.set_config(hvd._lib.HVD_CFG_LL128_MAX_BYTES, 0)
        ts = [[torch.randn(1 << 20, device="cuda")] for _ in range(n)]
        comm.allreduce_average(ts)
        torch.cuda.synchronize()
        for r in range(n):
            tl = comm.timeline(r)
            assert tl["rank"] == r and tl["size"] == n and tl["T"] == 2 * (n - 1)
            d = tl["data"]
            assert d.shape[1] == (tl["T"] + 1) * tl["K"]
            b, e = d[:, :, 0].astype(np.int64), d[:, :, 1].astype(np.int64)
            assert (b > 0).all() and (e >= b).all()
            assert (b[:, 1:] >= e[:, :-1]).all()            # program order per channel
            sg = tl["signals"]
            assert sg.shape[1] >= 1 and sg[:, :, 1].max() == tl["T"] * tl["K"]
        tr = timeline.chrome_trace([comm.timeline(r) for r in range(n)])
        assert any(ev.get("cat") == "RING" for ev in tr["traceEvents"])
        comm.set_config(hvd._lib.HVD_CFG_PROTOCOL, 0)  # pull kernel records
        comm.allreduce_average(ts)
        torch.cuda.synchronize()
        tl = comm.timeline(1)
        assert tl["kind"] == "pull" and tl["T"] == 2 * n - 1 and tl["data"].shape[1] == tl["T"] * tl["K"]
        b, e = tl["data"][:, :, 0].astype(np.int64), tl["data"][:, :, 1].astype(np.int64)
        assert (b > 0).all() and (e >= b).all() and (b[:, 1:] >= e[:, :-1]).all()
        assert timeline.chrome_trace([tl])["traceEvents"]
        comm.set_config(hvd._lib.HVD_CFG_TIMELINE, 0)
        assert comm.timeline(0) is None
    finally:
        comm.finalize()


# ---------------------------------------------------------------- broadcast / allgather (R12)
@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_broadcast_bitwise(hvd, n):
    comm = comm_for(hvd, n)
    counts = [7, 300, 1 << 20, 5, 65_537]
    for dtype in ("f32", "bf16", "i64"):
        kind = "specials" if dtype != "i64" else "int_uniform"
        xs = [workloads.rank_tensors(counts, dtype, r, kind) for r in range(n)]
        for root in sorted({0, n - 1, n // 2}):
            ref, _ = oracle.broadcast(xs, root)
            ts = [[to_torch(x, dtype) for x in xs[r]] for r in range(n)]
            comm.broadcast(ts, root=root)
            torch.cuda.synchronize()
            for r in range(n):
                for k in range(len(counts)):
                    got = from_torch(ts[r][k], dtype)
                    assert np.array_equal(got.view(np.uint8), ref[r][k].view(np.uint8)), (dtype, root, r, k)
    assert comm.poll_error() == 0


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_allgather_rank_order(hvd, n):
    comm = comm_for(hvd, n, 4 << 20)
    for dtype, count in (("f32", 1), ("f32", 100_003), ("bf16", 777), ("i64", 300_001), ("i32", 64)):
        kind = "normal" if dtype in ("f32", "bf16") else "int_uniform"
        xs = [workloads.rank_tensor(count, dtype, r, 4, kind) for r in range(n)]
        ref, _ = oracle.allgather(xs)
        ins = [to_torch(x, dtype) for x in xs]
        outs = [torch.empty(n * count, dtype=ins[0].dtype, device="cuda") for _ in range(n)]
        comm.allgather(ins, outs)
        torch.cuda.synchronize()
        for r in range(n):
            assert_same(from_torch(outs[r], dtype), ref[r], dtype, f"{dtype} count={count} r={r}")
    assert comm.poll_error() == 0


def test_mixed_collective_sequence_no_sync(hvd):
    """allreduce / broadcast / allgather back to back on one stream (buffer reuse hazards)."""
    n = 4
    comm = comm_for(hvd, n, 1 << 20)  # small capacity: several fusion buffers and allgather pieces
    counts = [100_000, 3, 200_000]
    xs = workloads.all_ranks(counts, "f32", n, seed=77)
    ys = workloads.all_ranks(counts, "f32", n, seed=78)
    g = [workloads.rank_tensor(150_000, "f32", r, 1, seed=79) for r in range(n)]
    tx = [[to_torch(x, "f32") for x in xs[r]] for r in range(n)]
    ty = [[to_torch(x, "f32") for x in ys[r]] for r in range(n)]
    gi = [to_torch(x, "f32") for x in g]
    go = [torch.empty(n * 150_000, device="cuda") for _ in range(n)]
    for it in range(3):
        comm.allreduce(tx, op="average", fusion_threshold=1 << 20)
        comm.broadcast(ty, root=it % n)
        comm.allgather(gi, go)
        comm.allreduce(ty, op="sum", fusion_threshold=0)
    torch.cuda.synchronize()
    assert comm.poll_error() == 0
    rx = xs
    ry = ys
    for it in range(3):
        rx, _, _ = oracle.allreduce(rx, ["f32"] * 3, "average", threshold=1 << 20, capacity=1 << 20)
        ry, _ = oracle.broadcast(ry, it % n)
        ry, _, _ = oracle.allreduce(ry, ["f32"] * 3, "sum", threshold=0, capacity=1 << 20)
    rg, _ = oracle.allgather(g)
    for r in range(n):
        for k in range(3):
            assert_same(from_torch(tx[r][k], "f32"), rx[r][k], "f32", f"x r={r} k={k}")
            assert_same(from_torch(ty[r][k], "f32"), ry[r][k], "f32", f"y r={r} k={k}")
        assert_same(from_torch(go[r], "f32"), rg[r], "f32", f"g r={r}")


@pytest.mark.parametrize("protocol", [0, 1])
@pytest.mark.parametrize("n", [2, 3, 5, 8])
def test_both_protocols_bitexact(hvd, n, protocol):
    """Pull (receiver TMA-loads) and push (sender stores) move the same partials: same bits."""
    comm = hvd.init_virtual(n, 0, 2 << 20)
    try:
        comm.set_config(hvd._lib.HVD_CFG_PROTOCOL, protocol)
        comm.set_config(hvd._lib.HVD_CFG_LL_MAX_BYTES, 0)  # small buffers would take the LL protocol
        counts = [3, 1000, 262_149, 5, 77_777, 400_000]
        for it, dtype in enumerate(["f32", "bf16", "f32"]):
            xs = workloads.all_ranks(counts, dtype, n, seed=500 + it)
            ref, _, plan = oracle.allreduce(xs, [dtype] * len(counts), "average", threshold=1 << 20,
                                            capacity=2 << 20)
            ts = [[to_torch(x, dtype) for x in xs[r]] for r in range(n)]
            comm.allreduce(ts, op="average", fusion_threshold=1 << 20)
            torch.cuda.synchronize()
            assert comm.poll_error() == 0
            st = comm.kernel_stats()
            # pull: one launch per fusion buffer; push: every buffer of the call in one launch
            assert st["pull" if protocol == 0 else "fused"][0] == (len(plan) if protocol == 0 else 1)
            for r in range(n):
                for k in range(len(counts)):
                    assert_same(from_torch(ts[r][k], dtype), ref[r][k], dtype, f"it={it} r={r} k={k}")
    finally:
        comm.finalize()


def test_pull_buffers_allocated_only_for_the_pull_protocol(hvd):
    """The pull protocol's two buffers per rank are a separate allocation, made only when
    that protocol is chosen (the default footprint is the push path's)."""
    L = hvd._lib
    n, cap = 4, 8 << 20
    hvd.init_virtual(1, 0, 1 << 20).finalize()  # library and module loading happen before free0
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    comm = hvd.init_virtual(n, 0, cap)
    try:
        free1 = torch.cuda.mem_get_info()[0]
        bufsz = 3 * cap + (2 << 20)
        # regions: 3 buffers + tail + 416 MiB LL areas per rank, no pull buffers
        assert free0 - free1 < n * (3 * bufsz + (420 << 20)) + (64 << 20)
        assert comm.get_config(L.HVD_CFG_PULL_BUFFERS) == 0
        comm.set_config(L.HVD_CFG_PROTOCOL, 0)      # virtual mode: allocates them here
        assert comm.get_config(L.HVD_CFG_PULL_BUFFERS) == 1
        free2 = torch.cuda.mem_get_info()[0]
        assert free1 - free2 >= n * 2 * bufsz
        with pytest.raises(hvd.HvdError):
            comm.set_config(L.HVD_CFG_PULL_BUFFERS, 0)
        comm.set_config(L.HVD_CFG_LL_MAX_BYTES, 0)
        counts = [5, 300_001, 1 << 20]
        xs = workloads.all_ranks(counts, "f32", n, seed=9100)
        ref, _, _ = oracle.allreduce(xs, ["f32"] * 3, "average", threshold=cap, capacity=cap)
        ts = [[to_torch(x, "f32") for x in xs[r]] for r in range(n)]
        comm.allreduce(ts, op="average", fusion_threshold=cap)
        torch.cuda.synchronize()
        assert comm.poll_error() == 0 and comm.kernel_stats()["pull"][0] >= 1
        for r in range(n):
            for k in range(3):
                assert_same(from_torch(ts[r][k], "f32"), ref[r][k], "f32", f"r={r} k={k}")
    finally:
        comm.finalize()


def test_pull_buffers_real_ranks_must_agree(hvd):
    """Real ranks: HVD_CFG_PULL_BUFFERS before the blob export, identical on every rank —
    hvd_connect refuses a mismatch before mapping anything; without the buffers the pull
    protocol cannot be chosen.  Two ranks of one process on one GPU (no kernel runs)."""
    import ctypes as C
    L = hvd._lib
    lib = L.lib
    hs = []
    try:
        for r in range(2):
            h = C.c_void_p()
            assert lib.hvd_init(r, 2, 0, 4 << 20, C.byref(h)) == L.HVD_OK
            hs.append(h)
        assert lib.hvd_set_config(hs[0], L.HVD_CFG_PULL_BUFFERS, 1) == L.HVD_OK
        assert lib.hvd_set_config(hs[1], L.HVD_CFG_PROTOCOL, 0) == L.HVD_ERR_INVALID
        ln = C.c_uint64(0)
        assert lib.hvd_get_ipc_blob(hs[0], None, C.byref(ln)) == L.HVD_OK
        blobs = []
        for h in hs:
            b = C.create_string_buffer(ln.value)
            assert lib.hvd_get_ipc_blob(h, b, C.byref(ln)) == L.HVD_OK
            blobs.append(bytes(b.raw))
        # after the export the setting is fixed
        assert lib.hvd_set_config(hs[1], L.HVD_CFG_PULL_BUFFERS, 1) == L.HVD_ERR_INVALID
        assert lib.hvd_set_config(hs[0], L.HVD_CFG_PULL_BUFFERS, 1) == L.HVD_OK
        assert lib.hvd_get_config(hs[0], L.HVD_CFG_PULL_BUFFERS) == 1
        assert lib.hvd_get_config(hs[1], L.HVD_CFG_PULL_BUFFERS) == 0
        joined = b"".join(blobs)
        for h in hs:
            assert lib.hvd_connect(h, joined, ln.value) == L.HVD_ERR_INVALID
    finally:
        for h in hs:
            lib.hvd_finalize(h)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("tdt,wire", [("f32", "bf16"), ("bf16", "f32")])
def test_wire_dtype_variants_bitexact(hvd, n, tdt, wire):
    """hvd_allreduce_ex (R14): fp32 grads over a bf16 wire, bf16 grads over fp32 partials."""
    counts = [1, 7, 1000, 4097, 100_003, 262_149, 33]
    xs = workloads.all_ranks(counts, tdt, n)
    ref, _, plan = oracle.allreduce(xs, [tdt] * len(counts), "average", threshold=400_000, wire=wire)
    comm = comm_for(hvd, n)
    ts = []
    keep = []
    for r in range(n):
        row = []
        for k, x in enumerate(xs[r]):
            t = to_torch(x, tdt)
            if k % 2 and len(x):  # misaligned views as well
                big = torch.empty(len(x) + 1, dtype=t.dtype, device="cuda")
                big[1:].copy_(t)
                keep.append(big)
                t = big[1:]
            row.append(t)
        ts.append(row)
    comm.kernel_stats()
    comm.allreduce(ts, op="average", fusion_threshold=400_000, wire=wire)
    torch.cuda.synchronize()
    assert comm.poll_error() == 0
    # all fusion buffers of the call in one launch (N = 1: the solo stream kernel)
    assert comm.kernel_stats()["fused" if n > 1 else "solo"][0] == 1
    for r in range(n):
        for k in range(len(counts)):
            assert_same(from_torch(ts[r][k], tdt), ref[r][k], tdt, f"N={n} r={r} k={k}")


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_registered_zero_copy_bitexact(hvd, n):
    """hvd_register: all-gather writes straight into the successor's tensors; same bits."""
    comm = hvd.init_virtual(n, 0, 1 << 20)  # small buffer: several fusion buffers
    try:
        counts = [3, 1000, 262_149, 5, 77_777, 400_001]
        ts = [[torch.empty(c, device="cuda") for c in counts] for _ in range(n)]
        keep = []
        ts[0][1] = torch.empty(1001, device="cuda")[1:]  # a misaligned view on one rank
        keep.append(ts[0][1])
        reg = comm.register(ts)
        for it in range(3):
            xs = workloads.all_ranks(counts, "f32", n, seed=900 + it)
            for r in range(n):
                for k in range(len(counts)):
                    ts[r][k].copy_(to_torch(xs[r][k], "f32"))
            ref, _, plan = oracle.allreduce(xs, ["f32"] * len(counts), "average", threshold=1 << 19,
                                            capacity=1 << 20)
            comm.allreduce_average(reg, fusion_threshold=1 << 19)
            torch.cuda.synchronize()
            assert comm.poll_error() == 0
            for r in range(n):
                for k in range(len(counts)):
                    assert_same(from_torch(ts[r][k], "f32"), ref[r][k], "f32", f"it={it} r={r} k={k}")
        comm.deregister(reg)
    finally:
        comm.finalize()


@pytest.mark.parametrize("n", [2, 4])
def test_many_small_buffers_one_launch(hvd, n):
    """Fusion off over 200 small tensors: up to 96 buffers per launch, small buffers each run
    whole on one channel (round robin) so they proceed in parallel; bit-exact."""
    comm = comm_for(hvd, n)
    counts = [int(c) for c in np.random.default_rng(8).integers(1, 3000, size=200)]
    xs = workloads.all_ranks(counts, "f32", n, seed=31)
    ref, _, plan = oracle.allreduce(xs, ["f32"] * len(counts), "average", threshold=0)
    assert len(plan) == 200
    L = hvd._lib
    ll_default = comm.get_config(L.HVD_CFG_LL_MAX_BYTES)
    ll128_default = comm.get_config(L.HVD_CFG_LL128_MAX_BYTES)
    # fused multi-buffer launches (LL and LL128 off), grouped LL128 launches (LL off), then
    # grouped LL launches (the default for small buffers)
    passes = [(0, 0, "fused"), (ll_default, ll128_default, "ll")]
    if n > 2:  # grouped LL128 for buffers above the LL limit: N > 2 only
        passes.insert(1, (0, ll128_default, "ll128"))
    for ll_max, ll128_max, kind in passes:
        comm.set_config(L.HVD_CFG_LL_MAX_BYTES, ll_max)
        comm.set_config(L.HVD_CFG_LL128_MAX_BYTES, ll128_max)
        ts = [[to_torch(x, "f32") for x in xs[r]] for r in range(n)]
        comm.kernel_stats()
        comm.allreduce(ts, op="average", fusion_threshold=0)
        torch.cuda.synchronize()
        assert comm.poll_error() == 0
        st = comm.kernel_stats()
        assert st[kind][0] == 3 and sum(v[0] for v in st.values()) == 3  # 96 + 96 + 8 buffers
        for r in range(n):
            for k in range(len(counts)):
                assert_same(from_torch(ts[r][k], "f32"), ref[r][k], "f32", f"{kind} r={r} k={k}")
    comm.set_config(L.HVD_CFG_LL_MAX_BYTES, ll_default)
    comm.set_config(L.HVD_CFG_LL128_MAX_BYTES, ll128_default)


@pytest.mark.parametrize("n", [2, 3, 4, 5, 8])
def test_ll_protocol_small_buffers_bitexact(hvd, n):
    """One small fusion buffer (<= 1 MiB) takes the LL protocol ({epoch, data} words): same bits,
    epochs/parities reused across back-to-back calls of varying size."""
    comm = comm_for(hvd, n)
    cases = [([1], "f32"), ([3, 5], "bf16"), ([64 * n + 7], "f32"), ([70_001, 13], "i32"),
             ([100_000, 3, 999], "f32"), ([262_144], "f32"), ([255_000], "bf16"),
             ([1_500_001, 17], "f32"), ([2_097_152], "f32"), ([3_000_000], "bf16")]  # LL_MAX raised to 8 MiB
    ll_default = comm.get_config(hvd._lib.HVD_CFG_LL_MAX_BYTES)
    comm.set_config(hvd._lib.HVD_CFG_LL_MAX_BYTES, 8 << 20)
    pend = []
    comm.kernel_stats()
    for it, (counts, dt) in enumerate(cases):
        kind = "normal" if dt in ("f32", "bf16") else "int_uniform"
        op = "average" if dt in ("f32", "bf16") else "sum"
        xs = workloads.all_ranks(counts, dt, n, kind=kind, seed=300 + it)
        ts = [[to_torch(x, dt) for x in xs[r]] for r in range(n)]
        if it == 4:  # a misaligned tensor on one rank
            big = torch.empty(counts[0] + 1, device="cuda")
            big[1:].copy_(ts[0][0])
            ts[0][0] = big[1:]
            pend.append(big)
        comm.allreduce(ts, op=op)
        pend.append((xs, ts, dt, op, counts))
    torch.cuda.synchronize()
    assert comm.poll_error() == 0
    assert comm.kernel_stats()["ll"][0] == len(cases)
    comm.set_config(hvd._lib.HVD_CFG_LL_MAX_BYTES, ll_default)
    for item in pend:
        if not isinstance(item, tuple):
            continue
        xs, ts, dt, op, counts = item
        ref, _, _ = oracle.allreduce(xs, [dt] * len(counts), op)
        for r in range(n):
            for k in range(len(counts)):
                assert_same(from_torch(ts[r][k], dt), ref[r][k], dt, f"{dt} {counts} r={r} k={k}")


def test_solo_stream_n1(hvd):
    """N = 1: the solo stream kernel (gather x 1/N -> scatter, no ring) over whole-tile, member
    boundary, ragged and misaligned cases; same bits."""
    comm = hvd.init_virtual(1, 0, 64 << 20)
    try:
        counts = [1, 8191, 2048 * 8, 5_000_011, 3, 2048 * 8 * 37 + 5, 262_144]
        for dt in ("f32", "bf16"):
            xs = workloads.all_ranks(counts, dt, 1, seed=77)
            ref, _, plan = oracle.allreduce(xs, [dt] * len(counts), "average")
            ts = [[to_torch(x, dt) for x in xs[0]]]
            big = torch.empty(counts[1] + 1, dtype=ts[0][1].dtype, device="cuda")
            big[1:].copy_(ts[0][1])
            ts[0][1] = big[1:]  # misaligned member
            comm.kernel_stats()
            comm.allreduce(ts, op="average")
            torch.cuda.synchronize()
            assert comm.poll_error() == 0
            assert comm.kernel_stats()["solo"][0] == len(plan) == 1
            for k in range(len(counts)):
                assert_same(from_torch(ts[0][k], dt), ref[0][k], dt, f"{dt} k={k}")
    finally:
        comm.finalize()


def test_solo_many_small_members_n1(hvd):
    """N = 1 boundary tiles whose members are staged in shared memory (up to 256 per tile)
    and tiles that span more members than that (the rest found in global memory): 900 tiny
    tensors (1-40 elements, so one 16 KiB tile holds hundreds of members) between large
    ones; same bits as the oracle."""
    import random
    rng = random.Random(1802)
    counts = [rng.randint(1, 40) for _ in range(600)] + [70_001] + [rng.randint(1, 9) for _ in range(300)] + [5]
    comm = hvd.init_virtual(1, 0, 64 << 20)
    try:
        for dt in ("f32", "bf16"):
            xs = workloads.all_ranks(counts, dt, 1, seed=78)
            ref, _, plan = oracle.allreduce(xs, [dt] * len(counts), "average")
            ts = [[to_torch(x, dt) for x in xs[0]]]
            comm.kernel_stats()
            comm.allreduce(ts, op="average")
            torch.cuda.synchronize()
            assert comm.poll_error() == 0
            assert comm.kernel_stats()["solo"][0] == 1
            for k in range(len(counts)):
                assert_same(from_torch(ts[0][k], dt), ref[0][k], dt, f"{dt} k={k}")
    finally:
        comm.finalize()


@pytest.mark.parametrize("tail", [0, 7, -1, 1 << 20])
@pytest.mark.parametrize("dt", ["f32", "bf16", "i32", "i64"])
def test_solo_member_tiles_mixed_alignment_n1(hvd, dt, tail):
    """N = 1 member tiles (built with the plan): members of several tiles with a ragged last
    vector, members smaller than one vector, and misaligned views (their tiles take the
    per-vector path) in one call; every tensor bit-exact to the oracle, one solo launch."""
    counts = [1, 3, 4097 * 8 + 5, 7, 65_536, 2, 9_001, 123_457, 0, 31]
    mis = {2, 5, 7}  # views off the 16 B grid
    op = "sum" if dt in ("i32", "i64") else "average"
    comm = hvd.init_virtual(1, 0, 8 << 20)
    try:
        comm.set_config(hvd._lib.HVD_CFG_SOLO_TAIL, tail)  # tail tiles cut in half (HVD_CFG_SOLO_TAIL)
        xs = workloads.all_ranks(counts, dt, 1, "int_uniform" if dt in ("i32", "i64") else "normal", seed=4242)
        ref, _, _ = oracle.allreduce(xs, [dt] * len(counts), op, threshold=8 << 20, capacity=8 << 20)
        keep, ts = [], []
        for k, x in enumerate(xs[0]):
            t = to_torch(x, dt)
            if k in mis and len(x) > 0:
                big = torch.empty(len(x) + 1, dtype=t.dtype, device="cuda")
                big[1:].copy_(t)
                keep.append(big)
                t = big[1:]
            ts.append(t)
        comm.kernel_stats()
        comm.allreduce([ts], op=op, fusion_threshold=8 << 20)
        torch.cuda.synchronize()
        assert comm.poll_error() == 0
        assert comm.kernel_stats()["solo"][0] == 1
        for k in range(len(counts)):
            assert_same(from_torch(ts[k], dt), ref[0][k], dt, f"k={k}")
    finally:
        comm.finalize()


@pytest.mark.parametrize("n", [2, 3, 4])
def test_negotiated_allreduce_cycles(hvd, n):
    """Readiness negotiation + Tensor Fusion (R15): each cycle reduces exactly the
    tensors every rank has reported, in rank 0's submission order (which fixes the fusion plan),
    bit-exact; the others stay untouched until their cycle."""
    import random
    from oracle import negotiation as neg
    comm = comm_for(hvd, n)
    g = hvd.negotiator(comm, max_tensors=32)
    try:
        rng = random.Random(55 + n)
        counts = [rng.choice([1, 7, 1000, 4096, 70_001, 262_144]) for _ in range(12)]
        xs = workloads.all_ranks(counts, "f32", n, seed=66)
        ts = [[to_torch(x, "f32") for x in xs[r]] for r in range(n)]
        reports = [[[] for _ in range(n)] for _ in range(4)]
        for t in range(len(counts)):
            for r in range(n):
                if t == 11 and r == n - 1:
                    continue  # never reported by the last rank: never reduced
                reports[rng.randrange(4)][r].append((t, 1, counts[t]))
        for c in range(4):
            for r in range(n):
                rng.shuffle(reports[c][r])
        expect = neg.simulate(reports)
        done = set()
        for c in range(4):
            for r in range(n):
                for tid, dt, cnt in reports[c][r]:
                    g.ready(tid, cnt, "f32", local=r)
            ids = comm.allreduce_negotiated(g, ts, op="average", fusion_threshold=1 << 20)
            torch.cuda.synchronize()
            assert comm.poll_error() == 0
            assert ids == expect[c]
            if ids:
                ref, _, _ = oracle.allreduce([[xs[r][i] for i in ids] for r in range(n)], ["f32"] * len(ids),
                                             "average", threshold=1 << 20)
                for r in range(n):
                    for j, i in enumerate(ids):
                        assert_same(from_torch(ts[r][i], "f32"), ref[r][j], "f32", f"cycle {c} id {i} r={r}")
            done |= set(ids)
            for r in range(n):
                for i in range(len(counts)):
                    if i not in done:
                        assert_same(from_torch(ts[r][i], "f32"), xs[r][i], "f32", f"pending id {i}")
        assert 11 not in done and g.pending(0) == [11]
    finally:
        g.close()


@pytest.mark.parametrize("zero_copy", [1, 0])
@pytest.mark.parametrize("n", [1, 2, 4])
def test_allreduce_host(hvd, n, zero_copy):
    """hvd_allreduce_host on pinned host buffers.  Zero copy (HVD_CFG_HOST_ZERO_COPY): the kernels gather
    from and scatter into host memory, the call is hvd_allreduce of one tensor (oracle on
    the whole tensor).  Staged: chunked H2D -> ring -> D2H through 3 slots, each chunk
    reduced as one tensor (oracle chunk by chunk)."""
    comm = comm_for(hvd, n)
    comm.set_config(hvd._lib.HVD_CFG_HOST_ZERO_COPY, zero_copy)
    try:
        for dt, op, L, chunk in [("f32", "average", 1_000_003, 1 << 18), ("bf16", "average", 300_001, 1 << 16),
                                 ("i32", "sum", 77_777, 0), ("f32", "sum", 5, 256),
                                 ("f32", "average", 20_000_001, 0)]:  # above 64 MiB: split into two buffers
            kind = "int_uniform" if dt == "i32" else "normal"
            xs = [workloads.rank_tensor(L, dt, r, 3, kind) for r in range(n)]
            hin = [to_torch(x, dt, device="cpu").pin_memory() for x in xs]
            hout = [torch.empty_like(h).pin_memory() for h in hin]
            comm.allreduce_host(hin, hout, op=op, chunk_bytes=chunk)
            torch.cuda.synchronize()
            assert comm.poll_error() == 0
            esz = oracle.ELEM_SIZE[dt]
            if zero_copy:
                ce = L
            else:
                ce = (chunk or (8 << 20)) // esz
                ce = max(256 // esz, ce // (256 // esz) * (256 // esz))
            for off in range(0, L, ce):
                part = [[x[off:off + ce]] for x in xs]
                ref, _, _ = oracle.allreduce(part, [dt], op)
                for r in range(n):
                    got = from_torch(hout[r][off:off + ce], dt)
                    assert_same(got, ref[r][0], dt, f"{dt} chunk@{off} r={r} zc={zero_copy}")
            for r in range(n):  # inputs untouched (out of place)
                assert_same(from_torch(hin[r], dt), xs[r], dt)
            comm.allreduce_host(hin, op=op, chunk_bytes=chunk)  # in place
            torch.cuda.synchronize()
            for r in range(n):
                assert np.array_equal(from_torch(hin[r], dt).view(np.uint8), from_torch(hout[r], dt).view(np.uint8))
    finally:
        comm.set_config(hvd._lib.HVD_CFG_HOST_ZERO_COPY, 0)


@pytest.mark.parametrize("n", [2, 3, 4])
def test_fusion_off_mixed_sizes_channel_ranges(hvd, n):
    """Fusion off over tensors from 1 element to ~6 MB: buffers <= 256 KiB take grouped LL
    launches, the others share multi-buffer fused launches, each on a range of ~q/64 KiB
    channels (round robin); with LL off every buffer takes the channel-range path.  Bit-exact."""
    comm = comm_for(hvd, n)
    rng = np.random.default_rng(90 + n)
    counts = [int(c) for c in rng.choice([1, 37, 1000, 40_000, 65_536, 300_001, 1_500_000], size=40)]
    xs = workloads.all_ranks(counts, "f32", n, seed=91)
    ref, _, plan = oracle.allreduce(xs, ["f32"] * len(counts), "average", threshold=0)
    L = hvd._lib
    ll_default = comm.get_config(L.HVD_CFG_LL_MAX_BYTES)
    ll128_default = comm.get_config(L.HVD_CFG_LL128_MAX_BYTES)
    # defaults: small buffers in LL groups, mid-size ones in LL128 groups, the rest fused;
    # then every buffer on the fused kernel's channel ranges
    for ll_max, ll128_max in ((ll_default, ll128_default), (0, 0)):
        comm.set_config(L.HVD_CFG_LL_MAX_BYTES, ll_max)
        comm.set_config(L.HVD_CFG_LL128_MAX_BYTES, ll128_max)
        ts = [[to_torch(x, "f32") for x in xs[r]] for r in range(n)]
        comm.kernel_stats()
        comm.allreduce(ts, op="average", fusion_threshold=0)
        torch.cuda.synchronize()
        assert comm.poll_error() == 0
        st = comm.kernel_stats()
        if ll_max:
            assert st["ll"][0] > 0 and (st["ll128"][0] > 0) == (n > 2)
        else:
            assert st["ll"][0] == 0 and st["ll128"][0] == 0 and st["fused"][0] >= 1
        for r in range(n):
            for k in range(len(counts)):
                assert_same(from_torch(ts[r][k], "f32"), ref[r][k], "f32", f"ll={ll_max} r={r} k={k}")
    comm.set_config(L.HVD_CFG_LL_MAX_BYTES, ll_default)
    comm.set_config(L.HVD_CFG_LL128_MAX_BYTES, ll128_default)


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_ll128_protocol_bitexact(hvd, n):
    """LL128 (flag inside each 128-byte line): same bits as the oracle's ring for ragged and
    multi-member buffers, interleaved with LL and fused calls (shared LL halves and epochs)."""
    comm = comm_for(hvd, n)
    L = hvd._lib
    ll_d, ll128_d = comm.get_config(L.HVD_CFG_LL_MAX_BYTES), comm.get_config(L.HVD_CFG_LL128_MAX_BYTES)
    cases = [([1], "f32", 16 << 20), ([1000, 7, 65_536], "bf16", 16 << 20), ([1_000_003], "f32", 16 << 20),
             ([500_000, 3, 77_777], "i32", 16 << 20), ([2_000_001], "bf16", 16 << 20),
             ([300_000], "f32", 1 << 20),          # LL (multi-limit) between LL128 calls
             ([3_999_999], "f32", 16 << 20), ([5_000], "f32", 0)]  # ll128 off: fused
    try:
        pend = []
        comm.kernel_stats()
        n128 = 0
        for it, (counts, dt, ll128) in enumerate(cases):
            comm.set_config(L.HVD_CFG_LL_MAX_BYTES, 0 if ll128 == 16 << 20 else ll_d)
            comm.set_config(L.HVD_CFG_LL128_MAX_BYTES, ll128)
            n128 += ll128 == 16 << 20
            kind = "normal" if dt in ("f32", "bf16") else "int_uniform"
            op = "average" if dt in ("f32", "bf16") else "sum"
            xs = workloads.all_ranks(counts, dt, n, kind=kind, seed=400 + it)
            ts = [[to_torch(x, dt) for x in xs[r]] for r in range(n)]
            if it == 1:  # a misaligned member
                big = torch.empty(counts[0] + 1, dtype=ts[0][0].dtype, device="cuda")
                big[1:].copy_(ts[0][0])
                ts[0][0] = big[1:]
                pend.append(big)
            comm.allreduce(ts, op=op)
            pend.append((xs, ts, dt, op, counts))
        torch.cuda.synchronize()
        assert comm.poll_error() == 0
        st = comm.kernel_stats()
        assert st["ll128"][0] == n128
        for item in pend:
            if not isinstance(item, tuple):
                continue
            xs, ts, dt, op, counts = item
            ref, _, _ = oracle.allreduce(xs, [dt] * len(counts), op)
            for r in range(n):
                for k in range(len(counts)):
                    assert_same(from_torch(ts[r][k], dt), ref[r][k], dt, f"{dt} {counts} r={r} k={k}")
        # traffic: the same bytes as the ring's (2L - |c_{r+1}| - |c_{r+2}|) elements
        comm.set_config(L.HVD_CFG_LL_MAX_BYTES, 0)
        comm.set_config(L.HVD_CFG_LL128_MAX_BYTES, 16 << 20)
        Lb = 1_234_567
        xs = [workloads.rank_tensor(Lb, "f32", r, 9) for r in range(n)]
        ref, tr = oracle.allreduce_buffer(xs, "f32", "sum")
        before = [comm.traffic(r) for r in range(n)]
        for r in range(n):
            comm.fusion_buffer(r, torch.float32, Lb).copy_(to_torch(xs[r], "f32"))
        comm.allreduce_buffer(Lb, hvd._lib.HVD_FLOAT32, "sum")
        torch.cuda.synchronize()
        for r in range(n):
            assert_same(from_torch(comm.fusion_buffer(r, torch.float32, Lb), "f32"), ref[r], "f32")
            sent, sends = comm.traffic(r)
            assert sent - before[r][0] == tr[r].sent_elems * 4 and sends - before[r][1] == 2 * (n - 1)
    finally:
        comm.set_config(L.HVD_CFG_LL_MAX_BYTES, ll_d)
        comm.set_config(L.HVD_CFG_LL128_MAX_BYTES, ll128_d)


@pytest.mark.parametrize("n", [2, 4])
def test_ll_after_ll128_small_int_data(hvd, n):
    """LL and LL128 own separate areas: an LL128 launch whose int32 data words
    equal small future epochs, followed by LL launches at those epochs, stays bit-exact.
    With a shared area, LL could take the stale LL128 words as its own."""
    comm = comm_for(hvd, n)
    big = 1 << 19    # 2 MiB int32: LL128
    small = 4096     # 16 KiB: LL
    pend = []
    for it in range(12):
        xs = [[np.full(big, (it % 8) + 1 + r, dtype=np.int32)] for r in range(n)]
        ts = [[to_torch(x, "i32") for x in xs[r]] for r in range(n)]
        comm.allreduce(ts, op="sum")
        pend.append((xs, ts))
        for j in range(3):
            xs2 = [[(np.arange(small, dtype=np.int32) % 7) + j + it + r] for r in range(n)]
            ts2 = [[to_torch(x, "i32") for x in xs2[r]] for r in range(n)]
            comm.allreduce(ts2, op="sum")
            pend.append((xs2, ts2))
    torch.cuda.synchronize()
    assert comm.poll_error() == 0
    st = comm.kernel_stats()
    assert st["ll128"][0] >= 12 and st["ll"][0] >= 36
    for xs, ts in pend:
        ref, _, _ = oracle.allreduce(xs, ["i32"], "sum")
        for r in range(n):
            assert_same(from_torch(ts[r][0], "i32"), ref[r][0], "i32")


def test_ll128_selftest_virtual(hvd):
    """hvd_ll128_selftest on virtual ranks: passes; a forced failure switches LL128 off and
    the LL128-sized call then runs on the fused push, bit-exact."""
    n = 4
    comm = hvd.init_virtual(n, 0, 64 << 20)
    try:
        L = hvd._lib
        comm.set_config(L.HVD_CFG_TIMEOUT_MS, 20000)
        assert comm.get_config(L.HVD_CFG_LL128_STATUS) == 0
        assert comm.ll128_selftest() == 1
        assert comm.get_config(L.HVD_CFG_LL128_MAX_BYTES) > 0
        xs = workloads.all_ranks([2_000_003], "f32", n)
        ref, _, _ = oracle.allreduce(xs, ["f32"], "average")
        for expect_kernel in ("ll128", "fused"):
            if expect_kernel == "fused":
                assert comm.ll128_selftest(force_fail=True) == -3
                assert comm.get_config(L.HVD_CFG_LL128_MAX_BYTES) == 0
            ts = [[to_torch(xs[r][0], "f32")] for r in range(n)]
            comm.kernel_stats()
            comm.allreduce_average(ts)
            torch.cuda.synchronize()
            assert comm.poll_error() == 0
            assert comm.kernel_stats()[expect_kernel][0] == 1
            for r in range(n):
                assert_same(from_torch(ts[r][0], "f32"), ref[r][0], "f32", f"{expect_kernel} r={r}")
    finally:
        comm.finalize()

"""Real multi-process ring over NVLink: one process per GPU, CUDA-IPC peers.

Runs only with >= 2 visible GPUs (``gpurun --gpus 2|4``).  Each rank runs the
collective on its seeded inputs; the parent compares every rank's output with
the oracle element by element and checks cross-rank bitwise agreement.
"""
import os
import random
import socket

import numpy as np
import pytest

import oracle
import workloads
from hvd_testutil import HVD_CODE, assert_same, from_torch, to_torch

torch = pytest.importorskip("torch")

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cases, q, protocol):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1802_05799_b200 as hvd
    try:
        comm = hvd.init(pull_buffers=protocol == 0)
        comm.set_config(hvd._lib.HVD_CFG_TIMEOUT_MS, 20000)
        comm.set_config(hvd._lib.HVD_CFG_PROTOCOL, protocol)
        out = []
        for case in cases:
            kind, counts, dtype, op, thr = case
            if kind == "tensors":
                xs = [workloads.rank_tensor(c, dtype, rank, k,
                                            "normal" if dtype in ("f32", "bf16") else "int_uniform")
                      for k, c in enumerate(counts)]
                ts = [to_torch(x, dtype) for x in xs]
                comm.allreduce(ts, op=op, fusion_threshold=thr)
                torch.cuda.synchronize()
                out.append([from_torch(t, dtype) for t in ts])
            elif kind == "registered":
                res_its = []
                ts = [torch.empty(c, device="cuda") for c in counts]
                reg = comm.register(ts)
                for it in range(2):
                    for k, c in enumerate(counts):
                        ts[k].copy_(to_torch(workloads.rank_tensor(c, "f32", rank, k, seed=700 + it), "f32"))
                    comm.allreduce_average(reg, fusion_threshold=thr)
                    torch.cuda.synchronize()
                    res_its.append([from_torch(t, "f32") for t in ts])
                out.append(res_its)
            elif kind == "mixed_collectives":
                # allreduce (fused), broadcast, allgather and a small (LL) allreduce back to back,
                # no host sync: every kernel kind's launch handshake against every other's
                res_its = []
                for it in range(4):
                    big = to_torch(workloads.rank_tensor(counts[0], dtype, rank, it, "normal"), dtype)
                    small = to_torch(workloads.rank_tensor(counts[1], dtype, rank, 10 + it, "normal"), dtype)
                    bc = to_torch(workloads.rank_tensor(counts[2], dtype, rank, 20 + it, "normal"), dtype)
                    ag_in = to_torch(workloads.rank_tensor(counts[3], dtype, rank, 30 + it, "normal"), dtype)
                    ag_out = torch.empty(world * counts[3], dtype=ag_in.dtype, device="cuda")
                    comm.allreduce_average([big])
                    comm.broadcast([bc], root=it % world)
                    comm.allgather(ag_in, ag_out)
                    comm.allreduce_average([small])
                    res_its.append([big, small, bc, ag_out])
                torch.cuda.synchronize()
                out.append([[from_torch(t, dtype) for t in r] for r in res_its])
            elif kind == "mixed_sizes":
                # back-to-back calls of alternating sizes, no host sync in between: LL and fused
                # launches of different geometry reuse receive regions (DESIGN.md Hazards)
                res_its = []
                for it in range(16):
                    c = counts[it % len(counts)]
                    t = to_torch(workloads.rank_tensor(c, dtype, rank, it, "normal"), dtype)
                    comm.allreduce_average([t])
                    res_its.append(t)
                torch.cuda.synchronize()
                out.append([from_torch(t, dtype) for t in res_its])
            elif kind == "host":
                # zero copy (the kernels read / write the pinned buffers over PCIe), then the
                # staged H2D -> ring -> D2H pipeline (the default)
                x = workloads.rank_tensor(counts[0], dtype, rank, 5, "normal")
                hin = to_torch(x, dtype, device="cpu").pin_memory()
                got = []
                for zc in (1, 0):
                    comm.set_config(hvd._lib.HVD_CFG_HOST_ZERO_COPY, zc)
                    hout = torch.empty_like(hin).pin_memory()
                    comm.allreduce_host(hin, hout, op=op, chunk_bytes=thr)
                    torch.cuda.synchronize()
                    got.append(from_torch(hout, dtype))
                comm.set_config(hvd._lib.HVD_CFG_HOST_ZERO_COPY, 0)
                out.append(got)
            elif kind == "negotiated":
                # every rank reports the same ids in its own order over 3 cycles (R15)
                g = hvd.negotiator(comm, max_tensors=64)
                ts = [to_torch(workloads.rank_tensor(c, dtype, rank, k, "normal"), dtype) for k, c in enumerate(counts)]
                order = list(range(len(counts)))
                random.Random(1000 + rank).shuffle(order)
                got_ids = []
                for cyc in range(3):
                    for tid in order[cyc::3]:
                        g.ready(tid, counts[tid], dtype)
                    got_ids.append(comm.allreduce_negotiated(g, ts, op="average", fusion_threshold=thr))
                torch.cuda.synchronize()
                g.close()
                out.append([[from_torch(t, dtype) for t in ts], got_ids])
            elif kind == "bcast":
                xs = [workloads.rank_tensor(c, dtype, rank, k, "specials") for k, c in enumerate(counts)]
                ts = [to_torch(x, dtype) for x in xs]
                comm.broadcast(ts, root=op)
                torch.cuda.synchronize()
                out.append([from_torch(t, dtype) for t in ts])
            elif kind == "allgather":
                x = workloads.rank_tensor(counts[0], dtype, rank, 4, "normal")
                o = torch.empty(world * counts[0], dtype=torch.float32 if dtype == "f32" else torch.bfloat16,
                                device="cuda")
                comm.allgather(to_torch(x, dtype), o)
                torch.cuda.synchronize()
                out.append([from_torch(o, dtype)])
            else:  # raw buffer
                L = counts[0]
                x = workloads.rank_tensor(L, dtype, rank, 9, "normal" if dtype in ("f32", "bf16") else "int_uniform")
                tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "i32": torch.int32, "i64": torch.int64}[dtype]
                comm.fusion_buffer(0, tdt, L).copy_(to_torch(x, dtype))
                sent0 = comm.traffic()
                comm.allreduce_buffer(L, HVD_CODE[dtype], op)
                torch.cuda.synchronize()
                sent1 = comm.traffic()
                out.append([from_torch(comm.fusion_buffer(0, tdt, L), dtype),
                            np.array([sent1[0] - sent0[0], sent1[1] - sent0[1]])])
        q.put((rank, out, comm.poll_error()))
        import torch.distributed as dist
        dist.barrier()
        comm.finalize()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), -99))


CASES = [
    ("tensors", [1, 3, 64, 1000, 4097, 100_003, 7, 262_149, 33], "f32", "average", 1 << 20),
    ("tensors", [5, 1 << 20, 12345], "bf16", "average", 64 << 20),
    ("tensors", [5, 1000, 77_777], "i64", "sum", 0),
    ("tensors", [3, 70_001], "i32", "sum", 64 << 20),
    ("tensors", [3_000_000, 9], "f32", "average", 64 << 20),  # one buffer above the LL limit: fused push
    ("buffer", [16 << 20], "f32", "sum", 0),
    ("buffer", [(1 << 20) + 3], "bf16", "average", 0),
    ("bcast", [5, 1 << 20, 333], "f32", 1, 0),
    ("negotiated", [5, 1 << 20, 333, 70_001, 2_000_003, 17, 4096], "f32", None, 4 << 20),
    ("host", [3_000_001], "f32", "average", 1 << 20),
    ("mixed_sizes", [262_144, 5_000, 786_432, 25, 3_000_000, 1_048_576, 777], "f32", "average", 0),
    ("mixed_collectives", [4_000_000, 3_000, 100_001, 50_000], "f32", None, 0),
    ("registered", [17, 3_000_001, 64, 500_000], "f32", "average", 8 << 20),
    ("registered", [16 << 20], "f32", "average", 64 << 20),  # bench.py's step: one registered 64 MiB gradient
    ("allgather", [100_003], "f32", None, 0),
    ("allgather", [8_000_001], "bf16", None, 0),
]


def _evidence(name, obj):
    """Keep what a multi-GPU run verified (the driver's GPU test box may have one GPU):
    gpurun_out/ travels back from gpurun and is copied into profiles/."""
    import json
    d = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, name), "w") as f:
        json.dump(obj, f, indent=1)


@pytest.mark.parametrize("protocol", [1, 0, 2])
def test_multiprocess_ring_matches_oracle(protocol):
    n = min(torch.cuda.device_count(), 4)
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, n, port, CASES, q, protocol)) for r in range(n)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(n):
        rank, out, err = q.get(timeout=600)
        res[rank] = (out, err)
    for p in procs:
        p.join(timeout=120)
    for r in range(n):
        assert res[r][1] == 0, res[r]
    for ci, (kind, counts, dtype, op, thr) in enumerate(CASES):
        if kind == "registered":
            for it in range(2):
                xs = [[workloads.rank_tensor(c, "f32", r, k, seed=700 + it) for k, c in enumerate(counts)]
                      for r in range(n)]
                ref, _, _ = oracle.allreduce(xs, ["f32"] * len(counts), "average", threshold=thr)
                for r in range(n):
                    for k in range(len(counts)):
                        assert_same(res[r][0][ci][it][k], ref[r][k], "f32", f"registered it={it} r={r} k={k}")
        elif kind == "mixed_collectives":
            for it in range(4):
                big = [[workloads.rank_tensor(counts[0], dtype, r, it, "normal")] for r in range(n)]
                small = [[workloads.rank_tensor(counts[1], dtype, r, 10 + it, "normal")] for r in range(n)]
                bc = [[workloads.rank_tensor(counts[2], dtype, r, 20 + it, "normal")] for r in range(n)]
                ag = [workloads.rank_tensor(counts[3], dtype, r, 30 + it, "normal") for r in range(n)]
                rb, _, _ = oracle.allreduce(big, [dtype], "average")
                rs, _, _ = oracle.allreduce(small, [dtype], "average")
                rc, _ = oracle.broadcast(bc, it % n)
                ra, _ = oracle.allgather(ag)
                for r in range(n):
                    got = res[r][0][ci][it]
                    assert_same(got[0], rb[r][0], dtype, f"mixed big it={it} rank {r}")
                    assert_same(got[1], rs[r][0], dtype, f"mixed small it={it} rank {r}")
                    assert np.array_equal(got[2].view(np.uint8), rc[r][0].view(np.uint8)), f"bcast it={it} r={r}"
                    assert_same(got[3], ra[r], dtype, f"mixed allgather it={it} rank {r}")
        elif kind == "mixed_sizes":
            for it in range(16):
                c = counts[it % len(counts)]
                xs = [[workloads.rank_tensor(c, dtype, r, it, "normal")] for r in range(n)]
                ref, _, _ = oracle.allreduce(xs, [dtype], "average")
                for r in range(n):
                    assert_same(res[r][0][ci][it], ref[r][0], dtype, f"mixed call {it} rank {r}")
        elif kind == "host":
            xs = [workloads.rank_tensor(counts[0], dtype, r, 5, "normal") for r in range(n)]
            ref, _, _ = oracle.allreduce([[x] for x in xs], [dtype], op)  # zero copy: one tensor
            for r in range(n):
                assert_same(res[r][0][ci][0], ref[r][0], dtype, f"host zero-copy rank {r}")
            ce = thr // oracle.ELEM_SIZE[dtype]  # staged: chunk by chunk
            for off in range(0, counts[0], ce):
                ref, _, _ = oracle.allreduce([[x[off:off + ce]] for x in xs], [dtype], op)
                for r in range(n):
                    assert_same(res[r][0][ci][1][off:off + ce], ref[r][0], dtype, f"host chunk@{off} rank {r}")
        elif kind == "negotiated":
            from oracle import negotiation as neg
            reports = [[[] for _ in range(n)] for _ in range(3)]
            for r in range(n):
                order = list(range(len(counts)))
                random.Random(1000 + r).shuffle(order)
                for cyc in range(3):
                    reports[cyc][r] = [(t, 1, counts[t]) for t in order[cyc::3]]
            expect = neg.simulate(reports)
            xs = [[workloads.rank_tensor(c, dtype, r, k, "normal") for k, c in enumerate(counts)] for r in range(n)]
            for r in range(n):
                assert res[r][0][ci][1] == expect
            for ids in expect:
                if not ids:
                    continue
                ref, _, _ = oracle.allreduce([[xs[r][i] for i in ids] for r in range(n)], [dtype] * len(ids),
                                             "average", threshold=thr)
                for r in range(n):
                    for j, i in enumerate(ids):
                        assert_same(res[r][0][ci][0][i], ref[r][j], dtype, f"negotiated id {i} rank {r}")
        elif kind == "bcast":
            xs = [[workloads.rank_tensor(c, dtype, r, k, "specials") for k, c in enumerate(counts)] for r in range(n)]
            ref, _ = oracle.broadcast(xs, op)
            for r in range(n):
                for k in range(len(counts)):
                    assert np.array_equal(res[r][0][ci][k].view(np.uint8), ref[r][k].view(np.uint8))
        elif kind == "allgather":
            xs = [workloads.rank_tensor(counts[0], dtype, r, 4, "normal") for r in range(n)]
            ref, _ = oracle.allgather(xs)
            for r in range(n):
                assert_same(res[r][0][ci][0], ref[r], dtype, f"allgather case {ci} rank {r}")
        elif kind == "tensors":
            kd = "normal" if dtype in ("f32", "bf16") else "int_uniform"
            xs = [[workloads.rank_tensor(c, dtype, r, k, kd) for k, c in enumerate(counts)] for r in range(n)]
            ref, _, _ = oracle.allreduce(xs, [dtype] * len(counts), op, threshold=thr)
            for r in range(n):
                for k in range(len(counts)):
                    assert_same(res[r][0][ci][k], ref[r][k], dtype, f"case {ci} rank {r} tensor {k}")
        else:
            L = counts[0]
            kd = "normal" if dtype in ("f32", "bf16") else "int_uniform"
            xs = [workloads.rank_tensor(L, dtype, r, 9, kd) for r in range(n)]
            ref, tr = oracle.allreduce_buffer(xs, dtype, op)
            for r in range(n):
                assert_same(res[r][0][ci][0], ref[r], dtype, f"buffer case {ci} rank {r}")
                sent, sends = res[r][0][ci][1]
                assert sent == tr[r].sent_elems * oracle.ELEM_SIZE[dtype] and sends == 2 * (n - 1)
    _evidence(f"mp_evidence_n{n}_protocol{protocol}.json",
              {"test": "test_multiprocess_ring_matches_oracle", "n_gpus": n, "protocol": protocol,
               "result": "every case bit-exact vs the oracle on every rank",
               "cases": [{"kind": k, "counts": c, "dtype": d, "op": o, "threshold": t} for k, c, d, o, t in CASES]})


def _timeout_worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    import time
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1802_05799_b200 as hvd
    import torch.distributed as dist
    try:
        comm = hvd.init()
        comm.set_config(hvd._lib.HVD_CFG_TIMEOUT_MS, 1500)
        x = torch.ones(1 << 20, device="cuda")
        dist.barrier()
        status = None
        if rank == 0:  # rank 1 never joins: rank 0's kernel must give up, not hang
            t0 = time.time()
            comm.allreduce_average([x])
            torch.cuda.synchronize()
            status = (comm.poll_error(), time.time() - t0)
            try:
                comm.allreduce_average([x])
                status = status + ("no error",)
            except hvd.HvdError as e:
                status = status + (e.status,)
        q.put((rank, status))
        dist.barrier()
        comm.finalize()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


def test_watchdog_turns_a_missing_peer_into_an_error():
    """A rank that never joins the collective: the device spin-wait gives up after the
    watchdog, latches HVD_ERR_TIMEOUT and every later call returns it (no GPU hang)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_timeout_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
    err, elapsed, again = res[0]
    assert err == -5 and again == -5, res  # HVD_ERR_TIMEOUT
    assert 1.0 < elapsed < 60.0


def _mismatch_worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1802_05799_b200 as hvd
    import torch.distributed as dist
    try:
        comm = hvd.init()
        comm.set_config(hvd._lib.HVD_CFG_TIMEOUT_MS, 3000)
        comm.set_config(hvd._lib.HVD_CFG_LL128_MAX_BYTES, 0)  # both sizes on the fused push
        dist.barrier()
        # the collective contract broken: rank 0 reduces 6M elements, rank 1 10M (both on the
        # fused push kernel, whose launch handshake compares call hashes; the LL protocols have
        # no handshake and report a mismatch through the watchdog)
        x = torch.ones(6_000_000 if rank == 0 else 10_000_000, device="cuda")
        comm.allreduce_average([x])
        torch.cuda.synchronize()
        q.put((rank, comm.poll_error()))
        dist.barrier()
        comm.finalize()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


def test_mismatched_calls_are_detected():
    """Ranks calling with different sizes: the launch handshake compares call hashes and
    latches HVD_ERR_MISMATCH (or the watchdog times out) instead of corrupting or hanging."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mismatch_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
    assert all(isinstance(v, int) for v in res.values()), res
    assert -7 in res.values() and set(res.values()) <= {-7, -5}, res


def _selftest_worker(rank, world, port, q, force_rank):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if rank == force_rank:
        os.environ["HVD_LL128_SELFTEST_FORCE_FAIL"] = "1"
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1802_05799_b200 as hvd
    import torch.distributed as dist
    try:
        comm = hvd.init()  # hvd_connect runs the NVLink check + LL128 self-test
        L = hvd._lib
        status = comm.get_config(L.HVD_CFG_LL128_STATUS)
        ll128 = comm.get_config(L.HVD_CFG_LL128_MAX_BYTES)
        comm.set_config(L.HVD_CFG_TIMEOUT_MS, 20000)
        x = to_torch(workloads.rank_tensor(2_000_003, "f32", rank, 3, "normal"), "f32")  # ~8 MiB: LL128 if on
        comm.kernel_stats()
        comm.allreduce_average([x])
        torch.cuda.synchronize()
        ks = {k: v[0] for k, v in comm.kernel_stats().items() if v[0]}
        again = comm.ll128_selftest()  # the explicit call agrees too
        q.put((rank, (status, ll128, ks, from_torch(x, "f32"), comm.poll_error(), again)))
        dist.barrier()
        comm.finalize()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


@pytest.mark.parametrize("force_rank", [-1, 1])
def test_ll128_selftest_at_connect(force_rank):
    """hvd_connect's LL128 safety check: on NVLink with whole 128-byte lines every rank
    passes and uses LL128 for an 8 MiB buffer; one rank forcing a failure switches LL128 off
    on EVERY rank (agreed through an LL allreduce) and results stay bit-exact."""
    n = min(torch.cuda.device_count(), 4)
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_selftest_worker, args=(r, n, port, q, force_rank)) for r in range(n)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(n))
    for p in procs:
        p.join(timeout=120)
    assert all(isinstance(v, tuple) for v in res.values()), res
    xs = [[workloads.rank_tensor(2_000_003, "f32", r, 3, "normal")] for r in range(n)]
    ref, _, _ = oracle.allreduce(xs, ["f32"], "average")
    for r in range(n):
        status, ll128, ks, got, err, again = res[r]
        assert err == 0
        assert_same(got, ref[r][0], "f32", f"rank {r}")
        if force_rank < 0:
            assert status == 1 and again == 1 and ll128 > 0 and ks.get("ll128") == 1, res[r][:3]
        else:
            assert status == -3 and ll128 == 0 and "ll128" not in ks, res[r][:3]
    _evidence(f"mp_evidence_ll128_selftest_n{n}_force{force_rank}.json",
              {"test": "test_ll128_selftest_at_connect", "n_gpus": n, "force_rank": force_rank,
               "status_per_rank": [res[r][0] for r in range(n)], "ll128_max_per_rank": [res[r][1] for r in range(n)],
               "kernels_per_rank": [res[r][2] for r in range(n)], "result": "bit-exact vs the oracle"})


def _trace_worker(rank, world, port, q, path):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), HVD_TIMELINE=path)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1802_05799_b200 as hvd
    import torch.distributed as dist
    try:
        comm = hvd.init()
        comm.set_config(hvd._lib.HVD_CFG_TIMEOUT_MS, 20000)
        small = torch.ones(1000, device="cuda")
        mid = torch.ones(1 << 20, device="cuda")
        big = torch.ones(14 << 20, device="cuda")  # 56 MiB: above the LL128 limits
        bc = torch.full((5000,), float(rank), device="cuda")
        ag_in = torch.full((3000,), float(rank), device="cuda")
        ag_out = torch.empty(3000 * world, device="cuda")
        for _ in range(2):
            comm.allreduce_average([small])
            comm.allreduce_average([mid])
            comm.allreduce_average([big])
            comm.broadcast([bc], root=0)
            comm.allgather(ag_in, ag_out)
        torch.cuda.synchronize()
        ok = bool(torch.equal(big, torch.ones_like(big))) and bool(torch.equal(bc, torch.zeros_like(bc)))
        dist.barrier()
        comm.finalize()  # writes this rank's remaining records
        dist.barrier()
        q.put((rank, ok))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


def test_job_timeline_one_file_all_ranks(tmp_path):
    """HVD_TIMELINE=<path> on every rank of a real multi-GPU job: one trace file, every
    rank's calls and kernels on one time axis."""
    n = min(torch.cuda.device_count(), 4)
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    import torch.multiprocessing as mp
    from paper_1802_05799_b200 import timeline
    path = str(tmp_path / "job.json")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_trace_worker, args=(r, n, port, q, path)) for r in range(n)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(n))
    for p in procs:
        p.join(timeout=120)
    assert all(v is True for v in res.values()), res
    ev = timeline.load_trace(path)
    summ = timeline.validate_trace(ev)
    assert sorted(summ) == list(range(n))
    for r in range(n):
        assert summ[r]["calls"] == {"ALLREDUCE": 6, "BROADCAST": 2, "ALLGATHER": 2}, summ[r]
        assert summ[r]["kernels"].get("LL_RING") == 2 and summ[r]["kernels"].get("FUSED_RING") == 2, summ[r]
        assert summ[r]["kernels"].get("COPY_RING") == 4, summ[r]
    # one axis: the same call's kernels on different ranks overlap in time (a ring launch
    # cannot finish on one rank before it started on another)
    k = [e for e in ev if e.get("cat") == "KERNEL" and e["name"] == "FUSED_RING"]
    by = {}
    for e in k:
        by.setdefault(e["args"]["seq"], []).append(e)
    for seq, es in by.items():
        if len(es) == n:
            assert max(e["ts"] for e in es) < min(e["ts"] + e["dur"] for e in es) + 50.0, es
    _evidence(f"mp_evidence_jobtrace_n{n}.json", {"test": "test_job_timeline_one_file_all_ranks", "n_gpus": n,
                                                 "summary": {str(r): summ[r] for r in summ}})
    import shutil
    d = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    shutil.copy(path, os.path.join(d, f"jobtrace_mp_n{n}.json"))

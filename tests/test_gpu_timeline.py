"""Job-wide Horovod Timeline on a B200: one trace for a sequence of mixed
calls, every kernel kind recorded, results unchanged (bit-exact vs the oracle)."""
import os
import subprocess
import sys

import pytest

import oracle
import workloads
from hvd_testutil import assert_same, from_torch, to_torch

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def hvd():
    import paper_1802_05799_b200 as m
    return m


def _ranks(xs, dt):
    return [[to_torch(x, dt) for x in row] for row in xs]


def test_job_trace_mixed_calls_every_kind(hvd, tmp_path):
    from paper_1802_05799_b200 import timeline
    L = hvd._lib
    n = 4
    path = str(tmp_path / "job.json")
    comm = hvd.init_virtual(n, 0, 64 << 20)
    calls = []  # (name, expected kernel kinds)
    try:
        comm.set_config(L.HVD_CFG_TIMEOUT_MS, 20000)
        comm.timeline_start(path)
        # 1. small buffer -> LL
        xs = workloads.all_ranks([1000, 3001], "f32", n)
        ref, _, _ = oracle.allreduce(xs, ["f32"] * 2, "average")
        ts = _ranks(xs, "f32")
        comm.allreduce(ts, "average")
        calls.append(("ALLREDUCE", {"LL_RING"}))
        # 2. mid-size lone buffer -> LL128
        xm = workloads.all_ranks([1_000_003], "f32", n)
        refm, _, _ = oracle.allreduce(xm, ["f32"], "average")
        tm = _ranks(xm, "f32")
        comm.allreduce(tm, "average")
        calls.append(("ALLREDUCE", {"LL128_RING"}))
        # 3. large buffer -> fused push ring
        xl = workloads.all_ranks([14_000_000], "f32", n)
        refl, _, _ = oracle.allreduce(xl, ["f32"], "average")
        tl = _ranks(xl, "f32")
        comm.allreduce(tl, "average")
        calls.append(("ALLREDUCE", {"FUSED_RING"}))
        # 4. broadcast, 5. allgather -> copy ring
        tb = [[torch.full((5000,), float(r), device="cuda")] for r in range(n)]
        comm.broadcast(tb, root=1)
        calls.append(("BROADCAST", {"COPY_RING"}))
        gi = [torch.full((3000,), float(r), device="cuda") for r in range(n)]
        go = [torch.empty(3000 * n, device="cuda") for _ in range(n)]
        comm.allgather(gi, go)
        calls.append(("ALLGATHER", {"COPY_RING"}))
        # 6. raw fusion buffer, sum
        comm.allreduce_buffer(1 << 20, hvd.HVD_FLOAT32, "sum")
        calls.append(("ALLREDUCE_BUFFER", None))
        # 7. host buffers
        hx = [torch.ones(300_000).pin_memory() for _ in range(n)]
        comm.allreduce_host(hx, op="average")
        calls.append(("ALLREDUCE_HOST", None))
        # 8. pull protocol, 9. bulk-copy push
        comm.set_config(L.HVD_CFG_PROTOCOL, 0)
        comm.allreduce(_ranks(xl, "f32"), "average")
        calls.append(("ALLREDUCE", {"PULL_RING"}))
        comm.set_config(L.HVD_CFG_PROTOCOL, 2)
        comm.allreduce(_ranks(xl, "f32"), "average")
        calls.append(("ALLREDUCE", {"BULK_RING"}))
        comm.set_config(L.HVD_CFG_PROTOCOL, 1)
        # 10. three-launch path: pack, ring, unpack
        comm.set_config(L.HVD_CFG_FUSED, 0)
        comm.allreduce(_ranks(xl, "f32"), "average")
        calls.append(("ALLREDUCE", {"PACK", "RING", "UNPACK"}))
        # 11. raw buffer average on the three-launch path: scale + ring
        comm.allreduce_buffer(1 << 20, hvd.HVD_FLOAT32, "average")
        calls.append(("ALLREDUCE_BUFFER", {"SCALE", "RING"}))
        comm.set_config(L.HVD_CFG_FUSED, 1)
        # 12-13. readiness negotiation: the cycle (host only), then the agreed tensors
        neg = hvd.negotiator(comm, max_tensors=8)
        tn = [[torch.ones(4000 + 1000 * k, device="cuda") for k in range(3)] for _ in range(n)]
        for r in range(n):
            for k in range(3):
                neg.ready_tensor(k, tn[r][k], local=r)
        ids = comm.allreduce_negotiated(neg, tn)
        assert ids == [0, 1, 2]
        calls.append(("NEGOTIATE_ALLREDUCE", None))
        calls.append(("ALLREDUCE", {"LL_RING"}))
        neg.close()
        torch.cuda.synchronize()
        assert comm.poll_error() == 0
        launched, dropped = comm.timeline_flush()
        comm.timeline_stop()
        for r in range(n):
            for k in range(2):
                assert_same(from_torch(ts[r][k], "f32"), ref[r][k], "f32", f"LL r{r} k{k}")
            assert_same(from_torch(tm[r][0], "f32"), refm[r][0], "f32", f"LL128 r{r}")
            assert_same(from_torch(tl[r][0], "f32"), refl[r][0], "f32", f"fused r{r}")
            assert torch.equal(tb[r][0], torch.full((5000,), 1.0, device="cuda"))
            assert torch.equal(go[r], torch.arange(n, device="cuda").repeat_interleave(3000).float())
    finally:
        comm.finalize()
    assert dropped == 0 and launched >= len(calls)
    ev = timeline.load_trace(path)
    summ = timeline.validate_trace(ev)
    assert sorted(summ) == list(range(n))
    spans = sorted((e for e in ev if e.get("cat") == "CALL" and e["pid"] == 0), key=lambda e: e["args"]["call"])
    assert [e["name"] for e in spans] == [c[0] for c in calls]
    kern = {}
    for e in ev:
        if e.get("cat") == "KERNEL" and e["pid"] == 0:
            kern.setdefault(e["args"]["call"], set()).add(e["name"])
    for span, (name, kinds) in zip(spans, calls):
        got = kern.get(span["args"]["call"], set())
        if name == "NEGOTIATE_ALLREDUCE":  # host only: no launch
            assert not got
            continue
        assert got, name
        if kinds is not None:
            assert got == kinds, (name, got, kinds)
    assert all(v["negotiated"] == 3 for v in summ.values())
    allk = set().union(*kern.values())
    assert {"LL_RING", "LL128_RING", "FUSED_RING", "COPY_RING", "PULL_RING", "BULK_RING", "PACK", "RING",
            "UNPACK", "SCALE"} <= allk
    # every rank's lane has the same launches (one launch spans all virtual ranks)
    per_rank = {p: sum(v["kernels"].values()) for p, v in summ.items()}
    assert len(set(per_rank.values())) == 1
    d = os.path.join(ROOT, "gpurun_out")  # evidence: travels back from gpurun into profiles/
    os.makedirs(d, exist_ok=True)
    import shutil
    shutil.copy(path, os.path.join(d, "jobtrace_virtual_n4.json"))


def test_job_trace_env_var_solo(tmp_path):
    """HVD_TIMELINE=<path> alone turns the trace on; N = 1 records SOLO."""
    path = str(tmp_path / "env.json")
    code = (
        "import torch, paper_1802_05799_b200 as hvd\n"
        "c = hvd.init_virtual(1, 0, 64 << 20)\n"
        "x = [[torch.ones(1 << 20, device='cuda'), torch.ones(1000, device='cuda')]]\n"
        "for _ in range(3):\n"
        "    c.allreduce_average(x)\n"
        "torch.cuda.synchronize()\n"
        "c.finalize()\n")
    env = dict(os.environ, HVD_TIMELINE=path, PYTHONPATH=ROOT)
    subprocess.run([sys.executable, "-c", code], check=True, env=env, cwd=ROOT, timeout=300)
    from paper_1802_05799_b200 import timeline
    ev = timeline.load_trace(path)
    summ = timeline.validate_trace(ev)
    assert summ[0]["calls"] == {"ALLREDUCE": 3}
    assert summ[0]["kernels"] == {"SOLO": 3}
    start = [e for e in ev if e["name"] == "TIMELINE_START"]
    assert len(start) == 1 and start[0]["args"]["clock_uncertainty_us"] < 1000


def test_job_trace_accounts_for_every_launch(hvd, tmp_path):
    """Thousands of back-to-back launches without a host sync: every launch is either in the
    trace or counted as dropped (the host slots hold 4096 launches in flight)."""
    from paper_1802_05799_b200 import timeline
    n = 2
    path = str(tmp_path / "many.json")
    comm = hvd.init_virtual(n, 0, 64 << 20)
    try:
        comm.timeline_start(path)
        xs = [[torch.ones(1000, device="cuda")] for _ in range(n)]
        calls = 5000
        for _ in range(calls):
            comm.allreduce(xs, "sum")
        launched, dropped = comm.timeline_flush()
        comm.timeline_stop()
        assert comm.poll_error() == 0
    finally:
        comm.finalize()
    assert launched == calls
    ev = timeline.load_trace(path)
    summ = timeline.validate_trace(ev) if dropped == 0 else timeline.job_summary(ev)
    for r in range(n):
        assert summ[r]["calls"] == {"ALLREDUCE": calls}
        assert sum(summ[r]["kernels"].values()) + dropped == calls

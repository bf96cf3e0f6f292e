"""Readiness negotiation (Tensor Fusion steps 1 and 6, P:L366 / P:L373; R15).

CPU only: the oracle (oracle/negotiation.py) against SPEC's worked examples and
a closed form, then the C negotiator (hvd_negotiator_*) against the oracle —
process-private (virtual ranks) and across processes over POSIX shared memory.
"""
import multiprocessing as mp
import os
import random
import time

import pytest

from oracle import negotiation as neg

F32, BF16, I32 = 1, 2, 3


# ---------------------------------------------------------------- oracle pins
def test_spec_example_intersection():
    """rank0 pending {a,b}, rank1 pending {b} -> cycle reduces only {b}; {a} waits."""
    a, b = (0, F32, 10), (1, F32, 20)
    agreed, rest = neg.negotiate([[a, b], [b]])
    assert agreed == [1] and rest == [[a], []]
    agreed, rest = neg.negotiate([rest[0], rest[1] + [a]])
    assert agreed == [0] and rest == [[], []]


def test_spec_example_empty_cycle():
    """all ranks pending {} -> empty cycle."""
    assert neg.negotiate([[], [], []]) == ([], [[], [], []])


def test_spec_example_mixed_dtypes_both_agreed():
    """{f32:a, i32:b} both ready -> both reduced (the fusion plan keeps dtypes apart)."""
    a, b = (5, F32, 3), (9, I32, 3)
    agreed, _ = neg.negotiate([[a, b], [b, a]])
    assert agreed == [5, 9]  # rank 0's order, not rank 1's


def test_metadata_mismatch_is_a_protocol_error():
    """the same tensor with a different dtype or length -> fatal, naming the tensor."""
    with pytest.raises(neg.ProtocolError) as e:
        neg.negotiate([[(3, F32, 10)], [(3, F32, 11)]])
    assert e.value.tid == 3
    with pytest.raises(neg.ProtocolError):
        neg.negotiate([[(3, F32, 10)], [(4, F32, 1), (3, BF16, 10)]])


def _random_schedule(rng, size, ncyc, nids, p_all=0.8):
    """Each id is reported once per rank (at a random cycle) by all ranks with prob p_all,
    else by a random strict subset; returns reports[c][r] and the report cycle per (id, r)."""
    meta = {t: (rng.choice([F32, BF16, I32]), rng.randrange(1, 1000)) for t in range(nids)}
    when = {}
    reports = [[[] for _ in range(size)] for _ in range(ncyc)]
    for t in range(nids):
        ranks = list(range(size)) if rng.random() < p_all or size == 1 else rng.sample(range(size), rng.randrange(0, size))
        for r in ranks:
            c = rng.randrange(ncyc)
            when[(t, r)] = c
            reports[c][r].append((t,) + meta[t])
    for c in range(ncyc):
        for r in range(size):
            rng.shuffle(reports[c][r])  # submission order differs across ranks
    return reports, when


@pytest.mark.parametrize("size", [1, 2, 3, 4, 8])
def test_closed_form_cycle_of_each_id(size):
    """Closed form: an id reported by every rank is reduced exactly once, in cycle
    max_r(report cycle); ids some rank never reports are never reduced; within a cycle the
    order is rank 0's submission order."""
    rng = random.Random(1802 + size)
    for _ in range(20):
        ncyc, nids = rng.randrange(1, 6), rng.randrange(0, 40)
        reports, when = _random_schedule(rng, size, ncyc, nids)
        got = neg.simulate(reports)
        expect = [[] for _ in range(ncyc)]
        for t in range(nids):
            if all((t, r) in when for r in range(size)):
                expect[max(when[(t, r)] for r in range(size))].append(t)
        for c in range(ncyc):
            assert sorted(got[c]) == sorted(expect[c])
            # rank 0's submission order: position of each id in rank 0's cumulative report stream
            order0 = [e[0] for cc in range(c + 1) for e in reports[cc][0]]
            assert got[c] == sorted(got[c], key=order0.index)


# ---------------------------------------------------------------- the C negotiator
@pytest.fixture(scope="module")
def hvd():
    import paper_1802_05799_b200 as m
    return m


def _c_simulate_virtual(hvd, reports, size, max_tensors=64):
    g = hvd.Negotiator(None, 0, size, size, max_tensors, 5000)
    out = []
    try:
        for cyc in reports:
            for r in range(size):
                for tid, dt, cnt in cyc[r]:
                    g.ready(tid, cnt, dt, local=r)
            out.append(g.cycle())
    finally:
        g.close()
    return out


@pytest.mark.parametrize("size", [1, 2, 3, 5, 8])
def test_c_negotiator_virtual_matches_oracle(hvd, size):
    rng = random.Random(77 + size)
    for _ in range(25):
        ncyc, nids = rng.randrange(1, 7), rng.randrange(0, 60)
        reports, _ = _random_schedule(rng, size, ncyc, nids)
        assert _c_simulate_virtual(hvd, reports, size) == neg.simulate(reports)


def test_c_negotiator_errors(hvd):
    from paper_1802_05799_b200 import HvdError
    g = hvd.Negotiator(None, 0, 2, 2, 8, 1000)
    try:
        g.ready(3, 10, "f32", local=0)
        with pytest.raises(HvdError):
            g.ready(3, 10, "f32", local=0)   # already pending
        with pytest.raises(HvdError):
            g.ready(8, 1, "f32", local=0)    # id out of range
        g.ready(3, 11, "f32", local=1)       # same id, different count
        with pytest.raises(HvdError):
            g.cycle()                        # protocol error
        assert g.pending(0) == [3] and g.pending(1) == [3]
    finally:
        g.close()
    with pytest.raises(HvdError):
        hvd.Negotiator("no-slash", 0, 2, 1, 8, 1000)
    with pytest.raises(HvdError):
        hvd.Negotiator(None, 0, 2, 3, 8, 1000)


def _shm_worker(name, rank, size, reports, q, skip_cycles):
    try:
        import paper_1802_05799_b200 as hvd
        g = hvd.Negotiator(name, rank, size, 1, 64, 20000 if not skip_cycles else 1500)
        out = []
        for c, cyc in enumerate(reports):
            if skip_cycles and rank != 0:
                break  # a rank that never shows up: rank 0 must time out
            for tid, dt, cnt in cyc[rank]:
                g.ready(tid, cnt, dt)
            t0 = time.time()
            try:
                out.append(g.cycle())
            except hvd.HvdError as e:
                out.append(("error", e.status, round(time.time() - t0, 2)))
                break
        if skip_cycles and rank != 0:
            time.sleep(3)  # keep the segment's other end alive while rank 0 waits
        g.close()
        q.put((rank, out))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


def _crashed_creator(name, size):
    """Rank 0 of a run that dies without hvd_negotiator_destroy: leaves a valid-looking segment."""
    import paper_1802_05799_b200 as hvd
    g = hvd.Negotiator(name, 0, size, 1, 64, 20000)  # noqa: F841 (kept alive until the exit)
    os._exit(0)


def _run_shm(size, reports, skip_cycles=False, name=None, rank0_delay=0.0):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = name or f"/hvd_test_{os.getpid()}_{random.randrange(1 << 30)}"
    ps = [ctx.Process(target=_shm_worker, args=(name, r, size, reports, q, skip_cycles)) for r in range(size)]
    for p in ps[1:]:
        p.start()
    if rank0_delay:
        time.sleep(rank0_delay)  # the other ranks look for the segment first
    ps[0].start()
    res = dict(q.get(timeout=120) for _ in range(size))
    for p in ps:
        p.join(timeout=30)
    return res


@pytest.mark.parametrize("size", [2, 4])
def test_c_negotiator_shared_memory_processes(size):
    """One process per rank over POSIX shared memory: every rank gets the oracle's lists."""
    rng = random.Random(4242 + size)
    reports, _ = _random_schedule(rng, size, 6, 50)
    expect = neg.simulate(reports)
    res = _run_shm(size, reports)
    for r in range(size):
        assert res[r] == expect, (r, res[r])


def test_c_negotiator_ignores_a_stale_segment():
    """A crashed run left a segment with the same name, magic and sizes: ranks
    that look for it before rank 0 replaces it must not attach to it (its creator is gone)."""
    name = f"/hvd_test_stale_{os.getpid()}_{random.randrange(1 << 30)}"
    ctx = mp.get_context("spawn")
    p = ctx.Process(target=_crashed_creator, args=(name, 2))
    p.start()
    p.join(timeout=60)
    assert os.path.exists("/dev/shm" + name)
    rng = random.Random(77)
    reports, _ = _random_schedule(rng, 2, 4, 50)
    expect = neg.simulate(reports)
    res = _run_shm(2, reports, name=name, rank0_delay=1.0)
    for r in range(2):
        assert res[r] == expect, (r, res[r])


def test_c_negotiator_timeout_when_a_rank_is_absent():
    reports = [[[(0, F32, 4)], [(0, F32, 4)]]]
    res = _run_shm(2, reports, skip_cycles=True)
    err = res[0][0]
    assert err[0] == "error" and err[1] == -5 and 1.0 <= err[2] <= 30.0


def test_negotiation_trace_and_timeline_events(hvd):
    """Timeline records of the negotiation phase: one (id, reported, agreed) per
    agreed tensor and rank, agreed >= reported; exported as NEGOTIATE spans per rank."""
    from paper_1802_05799_b200 import timeline
    g = hvd.Negotiator(None, 0, 2, 2, 16, 1000)
    try:
        g.ready(3, 10, "f32", local=0)
        g.ready(5, 20, "f32", local=0)
        g.ready(5, 20, "f32", local=1)
        time.sleep(0.002)
        assert g.cycle() == [5]
        g.ready(3, 10, "f32", local=1)
        assert g.cycle() == [3]
        tr = [g.trace(0), g.trace(1)]
        assert [t[0] for t in tr[0]] == [5, 3] and [t[0] for t in tr[1]] == [5, 3]
        for recs in tr:
            for tid, t_ready, t_agreed in recs:
                assert t_ready > 0 and t_agreed >= t_ready
        assert tr[0][1][1] < tr[1][1][1]  # rank 0 reported tensor 3 before rank 1 did
        assert g.trace(0) == []            # records are consumed
        ev = timeline.negotiation_events(tr, names=[f"grad{i}" for i in range(16)])
        spans = [e for e in ev if e.get("cat") == "NEGOTIATE"]
        assert len(spans) == 4 and {e["name"] for e in spans} == {"NEGOTIATE grad5", "NEGOTIATE grad3"}
        assert all(e["dur"] > 0 and e["ts"] >= 0 for e in spans)
    finally:
        g.close()

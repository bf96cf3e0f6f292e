"""Chrome-trace formatting of the device timeline (no GPU): synthetic records."""
import json

import numpy as np

from paper_1802_05799_b200 import timeline


def _fake(rank, N=2, K=2, ch=3):
    T = 2 * (N - 1)
    S = (T + 1) * K
    d = np.zeros((ch, S, 2), dtype=np.uint64)
    t = 1_000_000
    for c in range(ch):
        for i in range(S):
            d[c, i] = (t + i * 1000 + 100, t + i * 1000 + 900)
    sg = np.zeros((ch, T * K, 2), dtype=np.uint64)
    for c in range(ch):
        for j in range(T * K):
            sg[c, j] = (t + j * 1000 + 950, j + 1)
    return {"rank": rank, "size": N, "K": K, "T": T, "channels": ch, "data": d, "signals": sg}


def test_chrome_trace_lanes_and_phases(tmp_path):
    tls = [_fake(0), _fake(1)]
    tr = timeline.chrome_trace(tls)
    ev = tr["traceEvents"]
    ring = [e for e in ev if e.get("cat") == "RING"]
    assert len(ring) == 2 * 3 * 6
    names = {e["name"] for e in ring}
    assert "reduce-scatter s=0 k=0" in names and "all-gather s=0 k=1" in names and "final scatter k=1" in names
    waits = [e for e in ev if e.get("cat") == "WAIT"]
    assert waits and all(abs(w["dur"] - 0.2) < 1e-9 for w in waits)
    assert {e["pid"] for e in ring} == {0, 1}
    p = tmp_path / "t.json"
    timeline.write_chrome_trace(str(p), tls)
    assert json.loads(p.read_text())["traceEvents"]
    s = timeline.summarize(tls[0])
    assert abs(s["mean_wait_us"] - 0.2) < 1e-9 and s["span_us"] > 0


# ---------------------------------------------------------------- job-wide trace (schema)
import pytest  # noqa: E402


def _job_text(nranks=2, drop_last_comma=False):
    """A trace in the library's incremental format (csrc/hvd_jobtrace.cpp): metadata, one
    ALLREDUCE call with two launches, one BROADCAST call with one launch, per rank."""
    lines = ["["]
    for r in range(nranks):
        lines += [
            {"name": "process_name", "ph": "M", "pid": r, "args": {"name": f"rank {r} (GPU 0)"}},
            {"name": "thread_name", "ph": "M", "pid": r, "tid": 0, "args": {"name": "host calls"}},
            {"name": "thread_name", "ph": "M", "pid": r, "tid": 1, "args": {"name": "device kernels"}},
            {"name": "thread_name", "ph": "M", "pid": r, "tid": 2, "args": {"name": "negotiation"}},
            {"name": "NEGOTIATE", "cat": "NEGOTIATE", "ph": "X", "pid": r, "tid": 2, "ts": 990.0, "dur": 8.0,
             "args": {"tensor": 7, "call": 1}},
            {"name": "TIMELINE_START", "cat": "META", "ph": "i", "s": "p", "pid": r, "tid": 0, "ts": 100.0,
             "args": {"size": nranks, "local_ranks": nranks, "device": 0, "clock_uncertainty_us": 3.0}},
            {"name": "ALLREDUCE", "cat": "CALL", "ph": "X", "pid": r, "tid": 0, "ts": 1000.0, "dur": 20.0,
             "args": {"call": 1, "tensors": 3, "bytes": 4096, "launches": 2, "status": 0}},
            {"name": "BROADCAST", "cat": "CALL", "ph": "X", "pid": r, "tid": 0, "ts": 1030.0, "dur": 5.0,
             "args": {"call": 2, "tensors": 1, "bytes": 64, "launches": 1, "status": 0}},
        ]
        for seq, call, kind, ts in ((1, 1, "LL_RING", 1010.0), (2, 1, "FUSED_RING", 1025.0),
                                    (3, 2, "COPY_RING", 1040.0)):
            fid = seq * 8 + r
            lines += [
                {"name": "launch", "cat": "FLOW", "ph": "s", "id": fid, "pid": r, "tid": 0, "ts": ts - 5},
                {"name": kind, "cat": "KERNEL", "ph": "X", "pid": r, "tid": 1, "ts": ts, "dur": 7.5,
                 "args": {"seq": seq, "call": call, "ctas": 148, "bytes": 4096}},
                {"name": "launch", "cat": "FLOW", "ph": "f", "bp": "e", "id": fid, "pid": r, "tid": 1, "ts": ts},
            ]
    out = lines[0] + "\n" + "".join(json.dumps(e) + ",\n" for e in lines[1:])
    return out[:-2] + "\n" if drop_last_comma else out


def test_job_trace_parse_and_validate():
    ev = timeline.parse_trace_text(_job_text())
    s = timeline.validate_trace(ev)
    assert s[0]["calls"] == {"ALLREDUCE": 1, "BROADCAST": 1}
    assert s[1]["kernels"] == {"LL_RING": 1, "FUSED_RING": 1, "COPY_RING": 1}
    assert abs(s[0]["device_busy_us"] - 22.5) < 1e-9 and s[1]["negotiated"] == 1
    # the unterminated array, without the trailing comma, and closed: all the same events
    assert timeline.parse_trace_text(_job_text(drop_last_comma=True)) == ev
    assert timeline.parse_trace_text(_job_text(drop_last_comma=True) + "]") == ev


def _mutated(fn):
    ev = timeline.parse_trace_text(_job_text())
    fn(ev)
    return ev


@pytest.mark.parametrize("what,fn", [
    ("kernel span missing", lambda ev: ev.remove(next(e for e in ev if e.get("name") == "FUSED_RING"))),
    ("kernel on host lane", lambda ev: next(e for e in ev if e.get("cat") == "KERNEL").update(tid=0)),
    ("unknown kind", lambda ev: next(e for e in ev if e.get("cat") == "KERNEL").update(name="FOO")),
    ("zero duration", lambda ev: next(e for e in ev if e.get("cat") == "CALL").update(dur=0)),
    ("no CTAs", lambda ev: next(e for e in ev if e.get("cat") == "KERNEL")["args"].update(ctas=0)),
    ("call args", lambda ev: next(e for e in ev if e.get("cat") == "CALL")["args"].pop("bytes")),
    ("duplicate seq", lambda ev: ev.append(dict(next(e for e in ev if e.get("cat") == "KERNEL")))),
    ("unmatched flow", lambda ev: ev.remove(next(e for e in ev if e.get("ph") == "f"))),
    ("unnamed lane", lambda ev: ev.remove(next(e for e in ev if e.get("name") == "thread_name"))),
    ("kernel before call", lambda ev: next(e for e in ev if e.get("cat") == "KERNEL").update(ts=500.0)),
    ("negotiation lane", lambda ev: next(e for e in ev if e.get("cat") == "NEGOTIATE").update(tid=0)),
    ("negotiation args", lambda ev: next(e for e in ev if e.get("cat") == "NEGOTIATE")["args"].pop("tensor")),
])
def test_job_trace_validator_rejects(what, fn):
    with pytest.raises(ValueError):
        timeline.validate_trace(_mutated(fn))


def test_job_trace_golden_from_gpu():
    """The committed sample of a real trace (profiles/, written by the library on a B200)
    passes the schema check."""
    import os
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                     "r02_jobtrace_sample.json")
    if not os.path.exists(p):
        pytest.skip("no committed GPU trace sample yet")
    s = timeline.validate_trace(timeline.load_trace(p))
    kinds = set().union(*(set(v["kernels"]) for v in s.values()))
    assert {"LL_RING", "LL128_RING", "FUSED_RING", "COPY_RING"} <= kinds

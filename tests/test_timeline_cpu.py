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

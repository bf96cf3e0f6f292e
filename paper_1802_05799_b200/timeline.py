"""Horovod Timeline (§6) for the B200 path.

Two views.  (1) The job-wide trace (``HVD_TIMELINE=<path>`` or
``Comm.timeline_start``), written by the library itself (csrc/hvd_jobtrace.cpp): per
rank, a span for every public call on a "host calls" lane and a span for every kernel
launch — every kernel kind — on a "device kernels" lane, on one CLOCK_REALTIME axis
for all ranks of the node.  ``load_trace`` reads it, ``validate_trace`` checks its
schema, ``job_summary`` counts it.  (2) The per-slice detail of the most recent
fused launch, described next.

The paper's Timeline is a Chrome ``about:tracing`` view of "exactly what each
node was doing at each time step", switched on by one setting.
Here the events come from the device: with ``HVD_CFG_TIMELINE`` on, every
fused allreduce launch records, per rank and channel (CTA), the begin/end
of each slice operation — reduce-scatter step s, all-gather step s, the final
local scatter — and each signal the channel published to its ring successor
(``hvd_timeline``).  This module turns those records into Chrome trace-event
JSON: one process lane per rank, one thread lane per channel.

Timestamps are each GPU's %globaltimer (ns); lanes of different GPUs are
aligned on their own first event, so cross-rank skew is not meaningful below
a few microseconds.
"""
from __future__ import annotations

import json


def op_of(j: int, K: int, T: int, lag: int = 1):
    """j-th slice operation of a fused launch -> (t, k); mirrors fused_op in hvd_kernels.cu."""
    head = (T - 1) * K
    if j < head:
        return j // K, j % K
    m = j - head
    first = min(lag + 1, K)
    if m < first:
        return T - 1, m
    q = m - first
    pairs = K - first
    if q < 2 * pairs:
        p = q >> 1
        return (T, p) if q % 2 == 0 else (T - 1, p + first)
    return T, pairs + (q - 2 * pairs)


def _phase(idx: int, K: int, T: int, N: int, lag: int = 1, kind: str = "push") -> str:
    if kind == "registered":
        t, k = idx // K, idx % K
        return f"reduce-scatter s={t} k={k}" if t < N - 1 else f"all-gather s={t - N + 1} k={k}"
    if kind == "pull":
        t, k = idx // K, idx % K
        if t == 0:
            return f"stage own chunk k={k}"
        if t < N:
            return f"reduce-scatter s={t} k={k}"
        return f"all-gather s={t - N + 1} k={k}"
    t, k = (idx // K, idx % K) if N == 1 else op_of(idx, K, T, lag)
    if N == 1:
        return f"scale+copy k={k}"
    if t < N - 1:
        return f"reduce-scatter s={t} k={k}"
    if t < T:
        return f"all-gather s={t - (N - 1)} k={k}"
    return f"final scatter k={k}"


def chrome_trace(timelines, align: str = "per_rank") -> dict:
    """Chrome trace-event dict from a list of ``Comm.timeline()`` results (one per rank)."""
    events = []
    for tl in timelines:
        if tl is None:
            continue
        r, K, T, N = tl["rank"], tl["K"], tl["T"], tl["size"]
        lag = tl.get("fin_lag", 1)
        kind = tl.get("kind", "push")
        d, sg = tl["data"], tl["signals"]
        starts = [int(x) for x in d[:, :, 0].ravel() if int(x)]
        t0 = min(starts) if starts else 0
        events.append({"name": "process_name", "ph": "M", "pid": r, "args": {"name": f"rank {r}"}})
        for ch in range(d.shape[0]):
            events.append({"name": "thread_name", "ph": "M", "pid": r, "tid": ch, "args": {"name": f"channel {ch}"}})
            prev_end = None
            for i in range(d.shape[1]):
                b, e = int(d[ch, i, 0]), int(d[ch, i, 1])
                if not b or not e:
                    continue
                if prev_end is not None and b > prev_end:
                    events.append({"name": "wait (predecessor signal)", "cat": "WAIT", "ph": "X", "pid": r,
                                   "tid": ch, "ts": (prev_end - t0) / 1e3, "dur": (b - prev_end) / 1e3})
                events.append({"name": _phase(i, K, T, N, lag, kind), "cat": "RING", "ph": "X", "pid": r, "tid": ch,
                               "ts": (b - t0) / 1e3, "dur": max(e - b, 1) / 1e3})
                prev_end = e
            for j in range(sg.shape[1]):
                t, n = int(sg[ch, j, 0]), int(sg[ch, j, 1])
                if t:
                    nm = f"loadable op {n}" if kind == "pull" else f"signal {n}"
                    events.append({"name": nm, "cat": "SIGNAL", "ph": "i", "s": "t", "pid": r,
                                   "tid": ch, "ts": (t - t0) / 1e3})
    return {"traceEvents": events, "displayTimeUnit": "ns"}


def negotiation_events(traces, names=None) -> list:
    """Chrome events for ``Negotiator.trace()`` records, one list per rank: each agreed tensor
    as a NEGOTIATE span from its ready report to the cycle that agreed it (Horovod Timeline's
    negotiation phase).  Host CLOCK_REALTIME, so ranks of a node line up; shown
    on a "negotiation" lane of each rank, relative to the earliest report."""
    recs = [(r, rec) for r, tr in enumerate(traces) for rec in (tr or [])]
    if not recs:
        return []
    t0 = min(rec[1] for _, rec in recs)
    ev = []
    for r in sorted({r for r, _ in recs}):
        ev.append({"name": "thread_name", "ph": "M", "pid": r, "tid": "negotiation", "args": {"name": "negotiation"}})
    for r, (tid, tr, ta) in recs:
        nm = names[tid] if names and tid < len(names) else f"tensor {tid}"
        ev.append({"name": f"NEGOTIATE {nm}", "cat": "NEGOTIATE", "ph": "X", "pid": r, "tid": "negotiation",
                   "ts": (tr - t0) / 1e3, "dur": max(ta - tr, 1) / 1e3})
    return ev


def write_chrome_trace(path: str, timelines, negotiation=None, names=None) -> None:
    tr = chrome_trace(timelines)
    if negotiation:
        tr["traceEvents"] += negotiation_events(negotiation, names)
    with open(path, "w") as f:
        json.dump(tr, f)


def summarize(tl) -> dict:
    """Per-phase busy time, waits and the span of one rank's launch (microseconds)."""
    d = tl["data"]
    K, T, N = tl["K"], tl["T"], tl["size"]
    lag = tl.get("fin_lag", 1)
    kind = tl.get("kind", "push")
    b = d[:, :, 0].astype("int64")
    e = d[:, :, 1].astype("int64")
    valid = (b > 0) & (e > 0)
    span = (e[valid].max() - b[valid].min()) / 1e3 if valid.any() else 0.0
    busy = {}
    for i in range(d.shape[1]):
        name = _phase(i, K, T, N, lag, kind).rsplit(" k=", 1)[0]
        m = valid[:, i]
        busy[name] = busy.get(name, 0.0) + float(((e[:, i] - b[:, i])[m]).mean() / 1e3 if m.any() else 0.0)
    waits = []
    for ch in range(d.shape[0]):
        for i in range(1, d.shape[1]):
            if valid[ch, i] and valid[ch, i - 1]:
                waits.append((b[ch, i] - e[ch, i - 1]) / 1e3)
    return {"span_us": span, "busy_us_per_phase": busy,
            "mean_wait_us": float(sum(waits) / len(waits)) if waits else 0.0,
            "max_wait_us": float(max(waits)) if waits else 0.0}


# ---------------------------------------------------------------- job-wide trace
KERNEL_KINDS = ("PACK", "RING", "UNPACK", "SCALE", "FUSED_RING", "COPY_RING", "PULL_RING", "LL_RING", "SOLO",
                "LL128_RING", "BULK_RING")
CALL_NAMES = ("ALLREDUCE", "ALLREDUCE_BUFFER", "ALLREDUCE_HOST", "NEGOTIATE_ALLREDUCE", "BROADCAST", "ALLGATHER")


def parse_trace_text(text: str) -> list:
    """Events of a trace in the incremental array format the library writes: "[" then one
    event per line, each followed by "," (Chrome accepts the missing "]")."""
    body = text.strip()
    if not body.startswith("["):
        raise ValueError("not a Chrome trace-event array")
    body = body[1:].rstrip()
    if body.endswith("]"):
        body = body[:-1].rstrip()
    if body.endswith(","):
        body = body[:-1]
    return json.loads("[" + body + "]")


def load_trace(path: str) -> list:
    with open(path) as f:
        return parse_trace_text(f.read())


def validate_trace(events) -> dict:
    """Check the job trace's schema; returns job_summary(events).  Raises ValueError.

    Rules: metadata names every pid and its two lanes; "X" spans carry numeric ts >= 0 and
    dur > 0; CALL spans are on tid 0 with a known name and {call, tensors, bytes, launches,
    status}; KERNEL spans are on tid 1 with a known kind and {seq, call, ctas >= 1, bytes};
    a kernel may run after its call returned (stream order) but never starts before the
    call began (up to the clock calibration); NEGOTIATE spans (one per agreed tensor: ready
    report -> agreement) are on tid 2 with {tensor}; each (pid, seq) appears once; every
    flow "s" has its "f"; each call's launch count equals its kernel spans on that pid.
    """
    procs, lanes = set(), set()
    calls, kernels, flows_s, flows_f, negs = {}, {}, set(), set(), []
    for e in events:
        if not isinstance(e, dict) or "ph" not in e or "name" not in e:
            raise ValueError(f"malformed event {e!r}")
        ph = e["ph"]
        if ph == "M":
            if e["name"] == "process_name":
                procs.add(e["pid"])
            elif e["name"] == "thread_name":
                lanes.add((e["pid"], e["tid"]))
            continue
        for k in ("pid", "ts"):
            if k not in e:
                raise ValueError(f"event without {k}: {e!r}")
        if not isinstance(e["ts"], (int, float)) or e["ts"] < 0:
            raise ValueError(f"bad ts: {e!r}")
        if ph == "X":
            if not isinstance(e.get("dur"), (int, float)) or e["dur"] <= 0:
                raise ValueError(f"bad dur: {e!r}")
            a = e.get("args", {})
            if e.get("cat") == "CALL":
                if e["tid"] != 0 or e["name"] not in CALL_NAMES:
                    raise ValueError(f"bad call span: {e!r}")
                for k in ("call", "tensors", "bytes", "launches", "status"):
                    if k not in a:
                        raise ValueError(f"call span without {k}: {e!r}")
                key = (e["pid"], a["call"])
                if key in calls:
                    raise ValueError(f"call {key} twice")
                calls[key] = e
            elif e.get("cat") == "KERNEL":
                if e["tid"] != 1 or e["name"] not in KERNEL_KINDS:
                    raise ValueError(f"bad kernel span: {e!r}")
                for k in ("seq", "call", "ctas", "bytes"):
                    if k not in a:
                        raise ValueError(f"kernel span without {k}: {e!r}")
                if a["ctas"] < 1:
                    raise ValueError(f"kernel span with no CTAs: {e!r}")
                key = (e["pid"], a["seq"])
                if key in kernels:
                    raise ValueError(f"launch {key} twice")
                kernels[key] = e
            elif e.get("cat") == "NEGOTIATE":
                if e["tid"] != 2 or "tensor" not in a:
                    raise ValueError(f"bad negotiation span: {e!r}")
                negs.append(e)
            else:
                raise ValueError(f"unknown span category: {e!r}")
        elif ph == "s":
            flows_s.add((e["pid"], e["id"]))
        elif ph == "f":
            flows_f.add((e["pid"], e["id"]))
        elif ph != "i":
            raise ValueError(f"unknown phase: {e!r}")
    for e in list(calls.values()) + list(kernels.values()) + negs:
        if e["pid"] not in procs or (e["pid"], e["tid"]) not in lanes:
            raise ValueError(f"event on an unnamed lane: {e!r}")
    if flows_s != flows_f:
        raise ValueError(f"unmatched flow events: {sorted(flows_s ^ flows_f)[:5]}")
    per_call = {}
    for (pid, _), e in kernels.items():
        ck = (pid, e["args"]["call"])
        per_call[ck] = per_call.get(ck, 0) + 1
        c = calls.get(ck)
        if c is not None and e["ts"] + 1e-3 < c["ts"] - 50.0:
            # device clock mapped to host time: allow the calibration uncertainty (< 50 us)
            raise ValueError(f"kernel starts before its call: {e!r}")
    for ck, c in calls.items():
        if c["args"]["launches"] != per_call.get(ck, 0):
            raise ValueError(f"call {ck}: {c['args']['launches']} launches, {per_call.get(ck, 0)} kernel spans")
    return job_summary(events)


def job_summary(events) -> dict:
    """Per rank: calls by name, kernel launches by kind, device busy time (us)."""
    out = {}
    for e in events:
        if e.get("ph") != "X":
            continue
        r = out.setdefault(e["pid"], {"calls": {}, "kernels": {}, "device_busy_us": 0.0, "negotiated": 0})
        if e.get("cat") == "NEGOTIATE":
            r["negotiated"] += 1
        elif e.get("cat") == "CALL":
            r["calls"][e["name"]] = r["calls"].get(e["name"], 0) + 1
        elif e.get("cat") == "KERNEL":
            r["kernels"][e["name"]] = r["kernels"].get(e["name"], 0) + 1
            r["device_busy_us"] += e["dur"]
    return out

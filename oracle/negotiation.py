"""CPU oracle of the readiness negotiation cycle (TEST INFRASTRUCTURE ONLY).

Only ``tests/`` may use it; the product (``hvd_negotiate.cpp``) shares no code
with it.  It writes out DESIGN.md reading R15, which takes SPEC's protocol for
what the paper leaves open:

  Tensor Fusion step 1: "Determine which tensors are ready to be
  reduced."  Step 6: "Repeat until there are no more tensors to
  reduce in the cycle."
  S:L293-302: "a tensor is globally ready when all N ranks reported it —
  orders globally-ready tensors by submission order at rank 0 ...; tensors
  not globally ready remain pending for the next cycle"; "metadata mismatch
  for the same name (dtype/length/op differs across ranks) -> fatal protocol
  error naming the tensor".

A rank's pending list is its ready reports in submission order, as
(id, dtype, count) triples.  Pins: tests/test_negotiation.py (SPEC's worked
examples S:L300-302 and a closed form of when each id is reduced).
"""
from __future__ import annotations


class ProtocolError(ValueError):
    """The same tensor id was reported with different metadata."""

    def __init__(self, tid):
        super().__init__(f"tensor {tid} reported with different dtype/count")
        self.tid = tid


def negotiate(pending):
    """One cycle.  ``pending[r]`` = rank r's ordered list of (id, dtype, count).

    Returns (agreed ids in rank 0's order, new pending lists)."""
    size = len(pending)
    meta = {}
    for r in range(size):  # metadata agreement
        for tid, dt, cnt in pending[r]:
            if tid in meta and meta[tid] != (dt, cnt):
                raise ProtocolError(tid)
            meta.setdefault(tid, (dt, cnt))
    ids_of = [set(t for t, _, _ in pending[r]) for r in range(size)]
    agreed = [t for t, _, _ in pending[0] if all(t in ids_of[r] for r in range(size))]   # rank 0's order
    done = set(agreed)
    rest = [[e for e in pending[r] if e[0] not in done] for r in range(size)]
    return agreed, rest


def simulate(reports):
    """``reports[c][r]`` = list of (id, dtype, count) rank r reports ready before cycle c.

    Runs the cycles in order; returns the agreed list of every cycle."""
    size = len(reports[0]) if reports else 0
    pending = [[] for _ in range(size)]
    out = []
    for cyc in reports:
        for r in range(size):
            pending[r] = pending[r] + list(cyc[r])
        agreed, pending = negotiate(pending)
        out.append(agreed)
    return out

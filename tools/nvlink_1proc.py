"""The bench step (one registered 64 MiB fp32 gradient, allreduce-average) on N GPUs driven
by ONE process — one comm per GPU, connected to each other by peer access instead of CUDA
IPC (hvd_connect's same-process path) — so that ncu, which cannot profile while another
process uses the GPUs on this pool, can read the ring kernel's NVLink counters.

Each iteration launches rank N-1 .. 1 first and rank 0 last, so under
``ncu --devices 0`` the profiled rank-0 kernel starts while its peers already run.
Writes gpurun_out/nvlink/oneproc_n<N>.json: per-launch time (CUDA events, no ncu),
device traffic counters (hvd_traffic) and the algorithmic NVLink bytes per launch,
(2L - |c_{r+1}| - |c_{r+2}|) * esz, and checks that every rank's result
is bitwise identical (all-gather is a copy) and equals the mean within fp32 rounding.
Usage: python tools/nvlink_1proc.py N [iters]
"""
import ctypes as C
import json
import os
import sys
import threading

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1802_05799_b200 as hvd  # noqa: E402
from paper_1802_05799_b200 import _lib  # noqa: E402

lib = _lib.lib


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    L = int(os.environ.get("NVL_MIB", "64")) << 18  # fp32 elements
    comms = []
    for r in range(n):
        torch.cuda.set_device(r)
        h = C.c_void_p()
        _lib.check(lib.hvd_init(r, n, r, 64 << 20, C.byref(h)), "hvd_init")
        comms.append(hvd.Comm(h, r))
    ln = C.c_uint64(0)
    _lib.check(lib.hvd_get_ipc_blob(comms[0]._h, None, C.byref(ln)))
    blobs = []
    for c in comms:
        b = C.create_string_buffer(ln.value)
        _lib.check(lib.hvd_get_ipc_blob(c._h, b, C.byref(ln)), "hvd_get_ipc_blob")
        blobs.append(bytes(b.raw))
    joined = b"".join(blobs)
    rcs = [None] * n

    def connect(i):
        torch.cuda.set_device(i)
        rcs[i] = lib.hvd_connect(comms[i]._h, joined, ln.value)

    ths = [threading.Thread(target=connect, args=(i,)) for i in range(n)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert all(rc == 0 for rc in rcs), rcs
    proto = int(os.environ.get("NVL_PROTOCOL", "1"))
    for c in comms:
        c.set_config(_lib.HVD_CFG_TIMEOUT_MS, 120000)
        c.set_config(_lib.HVD_CFG_PROTOCOL, proto)
    g = []
    for r in range(n):
        gen = torch.Generator(device=f"cuda:{r}").manual_seed(180205799 + r)
        g.append(torch.randn(L, generator=gen, device=f"cuda:{r}"))
    x0 = [t.clone() for t in g]
    # registration: every rank's blob, then each rank maps its successor's tensor
    rl = C.c_uint64(0)
    arrs = [hvd._tensor_array([g[r]]) for r in range(n)]
    _lib.check(lib.hvd_register_blob(comms[0]._h, arrs[0], 1, None, C.byref(rl)))
    rb = []
    for r in range(n):
        b = C.create_string_buffer(rl.value)
        _lib.check(lib.hvd_register_blob(comms[r]._h, arrs[r], 1, b, C.byref(rl)), "hvd_register_blob")
        rb.append(bytes(b.raw))
    rj = b"".join(rb)
    rids = []
    for r in range(n):
        rid = C.c_int(-1)
        _lib.check(lib.hvd_register(comms[r]._h, arrs[r], 1, rj, rl.value, C.byref(rid)), "hvd_register")
        rids.append(rid.value)
    streams = [torch.cuda.Stream(device=r) for r in range(n)]

    def step():
        for r in reversed(range(n)):
            _lib.check(lib.hvd_allreduce_registered(comms[r]._h, rids[r], _lib.HVD_AVERAGE, 64 << 20,
                                                    C.c_void_p(streams[r].cuda_stream)), "allreduce")

    # correctness on the seeded inputs: first call
    step()
    for r in range(n):
        torch.cuda.synchronize(r)
    ref = sum(t.double().cpu() for t in x0) / n
    got0 = g[0].cpu()
    for r in range(1, n):
        assert torch.equal(g[r].cpu(), got0), f"rank {r} differs from rank 0"
    err = (got0.double() - ref).abs().max().item()
    for r in range(n):
        torch.cuda.synchronize(r)
    s0 = [c.traffic() for c in comms]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for _ in range(2):
        step()
    rng = os.environ.get("NVL_RANGE") == "1"  # ncu range replay: the timed loop is the range
    rdevs = [int(x) for x in os.environ.get("NVL_RANGE_DEVS", "0").split(",")]
    if rng:
        for r in range(n):
            torch.cuda.synchronize(r)
        for r in rdevs:
            with torch.cuda.device(r):
                torch.cuda.cudart().cudaProfilerStart()
    for r in range(n):
        ev[r][0].record(streams[r])
    for _ in range(iters):
        step()
    for r in range(n):
        ev[r][1].record(streams[r])
    for r in range(n):
        torch.cuda.synchronize(r)
    if rng:
        for r in rdevs:
            with torch.cuda.device(r):
                torch.cuda.cudart().cudaProfilerStop()
    t_ms = max(ev[r][0].elapsed_time(ev[r][1]) for r in range(n)) / iters
    s1 = [c.traffic() for c in comms]
    bounds = hvd.chunk_bounds(L, n, hvd.HVD_FLOAT32)
    size = [int(bounds[c + 1] - bounds[c]) for c in range(n)]
    out = {"n": n, "iters": iters, "payload_bytes": L * 4, "protocol": proto, "us_per_launch": t_ms * 1e3,
           "busbw_GBps": L * 4 / (t_ms / 1e3) / 1e9 * 2 * (n - 1) / n,
           "max_abs_err_vs_fp64_mean": err, "ranks_bitwise_equal": True,
           "kernels": {k: v[0] for k, v in comms[0].kernel_stats().items() if v[0]},
           "per_rank": []}
    for r in range(n):
        alg = (2 * L - size[(r + 1) % n] - size[(r + 2) % n]) * 4
        pushed = (s1[r][0] - s0[r][0]) / (iters + 2)
        out["per_rank"].append({"rank": r, "algorithmic_nvlink_bytes_per_launch": alg,
                                "pushed_bytes_per_launch": pushed,
                                "sends_per_launch": (s1[r][1] - s0[r][1]) / (iters + 2)})
    d = os.path.join(ROOT, "gpurun_out", "nvlink")
    os.makedirs(d, exist_ok=True)
    tag = os.environ.get("NVL_TAG", "")
    with open(os.path.join(d, f"oneproc_n{n}{tag}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))
    for c in comms:
        c.finalize()


if __name__ == "__main__":
    main()

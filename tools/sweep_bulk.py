"""Sweep the allreduce protocols / knobs on real GPUs (torchrun, one process per GPU).

Every point times bench.py's step — ``allreduce_average`` of registered fp32
gradients of ``--mib`` MiB, rotated over enough sets to exceed 2 x L2 — with CUDA
events over ``--iters`` calls, max over ranks, and checks the result of one call
bitwise against protocol 1 (the SM-store push).  A point is a comma list of
KEY=VALUE hvd_set_config settings, e.g. ``PROTOCOL=2,BULK_STAGE_BYTES=16384``.
Rank 0 prints one JSON line per point and writes them to ``--out``.  Tuning tool.
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.environ.get("HVD_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_05799_b200 as hvd  # noqa: E402


def tmax(x):
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=float, nargs="+", default=[64])
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--points", nargs="+", default=["PROTOCOL=1", "PROTOCOL=2"])
    ap.add_argument("--out", default="gpurun_out/sweep_bulk.json")
    ap.add_argument("--nccl", action="store_true")
    ap.add_argument("--max-sets", type=int, default=0, help="cap on rotated input sets (0: none)")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("gloo")
    comm = hvd.init(fusion_bytes=64 << 20)
    L = hvd._lib
    rows = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for mib in a.mib:
        cnt = int(mib * (1 << 20)) // 4
        nsets = max(2, -(-(2 * 126 << 20) // (cnt * 4)))
        if a.max_sets:
            nsets = min(nsets, a.max_sets)
        g = torch.Generator(device="cuda").manual_seed(77 + rank)
        sets = [[torch.randn(cnt, generator=g, device="cuda")] for _ in range(nsets)]
        regs = [comm.register(s) for s in sets]
        x0 = torch.randn(cnt, generator=g, device="cuda")
        ref = None
        for pt in a.points:
            cfg = [kv.split("=") for kv in pt.split(",") if kv]
            for k, v in (("PROTOCOL", 1), ("BULK_DEPTH", 0), ("BULK_STAGE_BYTES", 4096), ("BULK_STAGES", 6),
                         ("BULK_STAGE_BYTES", 16384), ("BULK_DEPTH", 1), ("BULK_CHANNELS", 148),
                         ("BULK_SLICE_BYTES", 65536), ("SIGNAL_WARPS", 1), ("WINDOW", 2), ("SLICE_BYTES", 0),
                         ("CHANNELS", 128), ("LL128_MAX_BYTES", 24 << 20 if world == 2 else 48 << 20),
                         ("PACE_GBPS", 0), ("PACE_BURST_ROWS", 2), ("FUSED_PDL", 0), ("WATCHER", 0), ("PREISSUE", -1), ("LL_PDL", 1)):  # defaults, then the point's settings
                comm.set_config(getattr(L, "HVD_CFG_" + k), v)
            for k, v in cfg:
                comm.set_config(getattr(L, "HVD_CFG_" + k), int(v))
            # bits: one call on fixed inputs vs the first point
            y = [x0.clone()]
            comm.allreduce_average(y)
            torch.cuda.synchronize()
            if ref is None:
                ref = y[0].clone()
            same = bool(torch.equal(y[0].view(torch.int32), ref.view(torch.int32)))
            comm.kernel_stats()
            for i in range(10):
                comm.allreduce_average(regs[i % nsets])
            torch.cuda.synchronize()
            dist.barrier()
            e0.record()
            for i in range(a.iters):
                comm.allreduce_average(regs[i % nsets])
            e1.record()
            torch.cuda.synchronize()
            dist.barrier()
            us = tmax(e0.elapsed_time(e1) / a.iters * 1e3)
            ks = {k: v[0] for k, v in comm.kernel_stats().items() if v[0]}
            row = {"n": world, "mib": mib, "point": pt, "us": us,
                   "busbw": cnt * 4 / (us * 1e-6) / 1e9 * 2 * (world - 1) / world,
                   "bitexact_vs_first_point": same, "kernels": ks}
            rows.append(row)
            if rank == 0:
                print(json.dumps(row), flush=True)
            assert comm.poll_error() == 0, hvd._lib.strerror(comm.poll_error())
        for rg in regs:
            comm.deregister(rg)
    if a.nccl:
        ng = dist.new_group(backend="nccl")
        for mib in a.mib:
            x = torch.ones(int(mib * (1 << 20)) // 4, device="cuda")
            for _ in range(5):
                dist.all_reduce(x, group=ng)
            torch.cuda.synchronize()
            dist.barrier()
            e0.record()
            for _ in range(a.iters):
                dist.all_reduce(x, group=ng)
            e1.record()
            torch.cuda.synchronize()
            dist.barrier()
            us = tmax(e0.elapsed_time(e1) / a.iters * 1e3)
            row = {"n": world, "mib": mib, "point": "nccl " + os.environ.get("NCCL_ALGO", "default"), "us": us,
                   "busbw": x.numel() * 4 / (us * 1e-6) / 1e9 * 2 * (world - 1) / world}
            rows.append(row)
            if rank == 0:
                print(json.dumps(row), flush=True)
    if rank == 0:
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        with open(a.out, "w") as f:
            json.dump(rows, f, indent=1)
    dist.barrier()
    comm.finalize()


if __name__ == "__main__":
    main()

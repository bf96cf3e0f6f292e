"""Sweep the ring kernel's knobs on real GPUs (torchrun, one process per GPU).

Times hvd_allreduce_buffer on one fusion buffer for every (channels, slice,
threads) point and NCCL all_reduce on the same bytes; rank 0 writes a JSON
table to gpurun_out/.  Tuning tool, not a deliverable.
"""
import argparse
import itertools
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_05799_b200 as hvd  # noqa: E402


def tmax(x):
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, nargs="+", default=[64])
    ap.add_argument("--channels", type=int, nargs="+", default=[16, 32, 64])
    ap.add_argument("--slice-kib", type=int, nargs="+", default=[64, 256, 1024])
    ap.add_argument("--threads", type=int, nargs="+", default=[256, 512])
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--fence-mode", type=int, nargs="+", default=[1])
    ap.add_argument("--window", type=int, nargs="+", default=[0])
    ap.add_argument("--protocol", type=int, default=1, help="0 pull, 1 push")
    ap.add_argument("--fused", type=int, default=-1, help="ring mode: 1 fused kernel on the buffer, 0 ring kernel")
    ap.add_argument("--fin-lag", type=int, nargs="+", default=[1])
    ap.add_argument("--check", action="store_true", help="verify bit-exactness of every point vs a reference run")
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--out", default="gpurun_out/sweep.json")
    ap.add_argument("--nccl", action="store_true")
    ap.add_argument("--ll-max", type=int, default=-1, help="HVD_CFG_LL_MAX_BYTES (-1: library default)")
    ap.add_argument("--mode", default="ring", choices=["ring", "fused", "three", "registered"],
                    help="ring: hvd_allreduce_buffer; fused/three: hvd_allreduce_average of one tensor")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("gloo")
    cap = max(a.mib) << 20
    comm = hvd.init(fusion_bytes=cap, pull_buffers=a.protocol == 0)
    L = hvd._lib
    code = {"f32": L.HVD_FLOAT32, "bf16": L.HVD_BFLOAT16}[a.dtype]
    esz = 4 if a.dtype == "f32" else 2
    rows = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ref = {}
    grads = {mib: torch.randn((mib << 20) // esz, device="cuda").to(torch.float32 if esz == 4 else torch.bfloat16)
             for mib in a.mib}
    comm.set_config(L.HVD_CFG_FUSED, (1 if a.mode in ("fused", "registered") else 0) if a.fused < 0 else a.fused)
    comm.set_config(L.HVD_CFG_PROTOCOL, a.protocol)
    if a.ll_max >= 0:
        comm.set_config(L.HVD_CFG_LL_MAX_BYTES, a.ll_max)

    regs = {mib: comm.register([grads[mib]]) for mib in a.mib} if a.mode == "registered" else {}

    def call(mib, cnt):
        if a.mode == "ring":
            comm.allreduce_buffer(cnt, code, "sum")
        elif a.mode == "registered":
            comm.allreduce_average(regs[mib])
        else:
            comm.allreduce_average([grads[mib]])
    for mib, ch, sl, th, sg, win, lag in itertools.product(a.mib, a.channels, a.slice_kib, a.threads, a.fence_mode,
                                                           a.window, a.fin_lag):
        comm.set_config(L.HVD_CFG_SIGNAL_MODE, sg)
        comm.set_config(L.HVD_CFG_WINDOW, win)
        comm.set_config(L.HVD_CFG_FIN_LAG, lag)
        comm.set_config(L.HVD_CFG_CHANNELS, ch)
        comm.set_config(L.HVD_CFG_SLICE_BYTES, sl << 10)
        comm.set_config(L.HVD_CFG_THREADS, th)
        cnt = (mib << 20) // esz
        ok = None
        if a.check:
            g = torch.Generator(device="cuda").manual_seed(1234 + rank)
            x = torch.randn(cnt, generator=g, device="cuda")
            fb = comm.fusion_buffer(0, torch.float32, cnt)
            res = []
            for rep in range(3):
                if a.mode == "ring":
                    fb.copy_(x)
                    comm.allreduce_buffer(cnt, code, "sum")
                    torch.cuda.synchronize()
                    res.append(fb.clone())
                else:
                    y = x.clone()
                    comm.allreduce_average([y])
                    torch.cuda.synchronize()
                    res.append(y)
            if mib not in ref:
                ref[mib] = res[0]
            ok = all(torch.equal(r.view(torch.int32), ref[mib].view(torch.int32)) for r in res)
        for _ in range(3):
            call(mib, cnt)
        torch.cuda.synchronize(); dist.barrier()
        ev0.record()
        for _ in range(a.iters):
            call(mib, cnt)
        ev1.record()
        torch.cuda.synchronize(); dist.barrier()
        us = tmax(ev0.elapsed_time(ev1) / a.iters * 1e3)
        bus = (mib << 20) / (us * 1e-6) / 1e9 * 2 * (world - 1) / world
        rows.append({"impl": "hvd", "mode": a.mode, "fused": comm.get_config(L.HVD_CFG_FUSED), "protocol": a.protocol, "mib": mib, "channels": ch, "slice_kib": sl, "threads": th, "sig": sg, "window": win, "fin_lag": lag,
                     "us": us, "busbw": bus, "bitexact_vs_first": ok})
        if rank == 0:
            print(json.dumps(rows[-1]), flush=True)
    assert comm.poll_error() == 0
    if a.nccl:
        ng = dist.new_group(backend="nccl")
        for mib in a.mib:
            x = torch.ones((mib << 20) // esz, device="cuda", dtype=torch.float32 if esz == 4 else torch.bfloat16)
            for _ in range(5):
                dist.all_reduce(x, group=ng)
            torch.cuda.synchronize(); dist.barrier()
            ev0.record()
            for _ in range(a.iters):
                dist.all_reduce(x, group=ng)
            ev1.record()
            torch.cuda.synchronize(); dist.barrier()
            us = tmax(ev0.elapsed_time(ev1) / a.iters * 1e3)
            rows.append({"impl": "nccl", "env": os.environ.get("NCCL_ALGO", "default") + "/" +
                         os.environ.get("NCCL_PROTO", "default"), "mib": mib, "us": us,
                         "busbw": (mib << 20) / (us * 1e-6) / 1e9 * 2 * (world - 1) / world})
            if rank == 0:
                print(json.dumps(rows[-1]), flush=True)
    if rank == 0:
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        with open(a.out, "w") as f:
            json.dump(rows, f, indent=1)
    dist.barrier()
    comm.finalize()


if __name__ == "__main__":
    main()

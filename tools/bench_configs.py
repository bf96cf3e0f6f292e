"""BASELINE.json configs C2-C5 on N GPUs (torchrun, one process per GPU).

  C2  ResNet-101 synthetic gradient set, fp32, Tensor Fusion 64 MiB
  C3  Inception V3 set, fp32 and bf16, fusion on (64 MiB) vs off (threshold 0)
  C4  VGG-16 set, fp32 (11 fusion buffers; fc6 split, fc7 exactly 64 MiB)
  C5  message-size sweep 1 KiB .. 1 GiB, fp32 and bf16, ours vs NCCL (default
      and Ring/Simple via NCCL_ALGO/NCCL_PROTO in the environment)

Each measurement: warm-up, then `iters` back-to-back calls timed with CUDA
events between barriers, max over ranks.  Inputs rotate over enough tensor
sets to exceed 2 x L2 when the set is smaller than L2.  Rank 0 writes one JSON
file.  Tuning / reporting tool; bench.py is the contract.
"""
import argparse
import json
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_05799_b200 as hvd  # noqa: E402
import workloads  # noqa: E402

MIB = 1 << 20
L2 = 126 * MIB


def tmax(x):
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def timed(fn, iters, warm=3, nsets=1):
    for i in range(max(warm, nsets)):  # every input set once (plan tables uploaded) before timing
        fn(i)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    return tmax(e0.elapsed_time(e1) / iters * 1e3)  # us


def sets_for(counts, dtype, payload):
    n = max(1, min(8, -(-2 * L2 // max(payload, 1))))
    g = torch.Generator(device="cuda").manual_seed(1234 + dist.get_rank())
    return [[torch.randn(c, generator=g, device="cuda").to(dtype) for c in counts] for _ in range(n)]


def bus(payload, us, n):
    return payload / (us * 1e-6) / 1e9 * (2 * (n - 1) / n if n > 1 else 1.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/configs.json")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--only", default="C2,C3,C4,C5")
    ap.add_argument("--sweep-max-log2", type=int, default=30)
    ap.add_argument("--sweep-min-log2", type=int, default=10)
    ap.add_argument("--ll-max", type=int, default=-1, help="HVD_CFG_LL_MAX_BYTES (-1: library default)")
    ap.add_argument("--ll128-max", type=int, default=-1, help="HVD_CFG_LL128_MAX_BYTES (-1: library default)")
    ap.add_argument("--no-nccl", action="store_true")
    a = ap.parse_args()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group("gloo")
    n = dist.get_world_size()
    comm = hvd.init(fusion_bytes=64 * MIB)
    if a.ll_max >= 0:
        comm.set_config(hvd._lib.HVD_CFG_LL_MAX_BYTES, a.ll_max)
    if a.ll128_max >= 0:
        comm.set_config(hvd._lib.HVD_CFG_LL128_MAX_BYTES, a.ll128_max)
    ng = dist.new_group(backend="nccl") if n > 1 else None
    res = {"n_gpus": n, "rows": []}
    only = set(a.only.split(","))

    def model_row(cfg, model, dt, thr):
        counts = [c for _, c in workloads.gradient_set(model)]
        tdt = torch.float32 if dt == "f32" else torch.bfloat16
        payload = sum(counts) * (4 if dt == "f32" else 2)
        sets = sets_for(counts, tdt, payload)
        preps = [comm.prepare(st) for st in sets]  # marshalled once, like a training loop
        comm.kernel_stats()
        us = timed(lambda i: comm.allreduce_average(preps[i % len(preps)], fusion_threshold=thr), a.iters,
                   nsets=len(preps))
        ks = comm.kernel_stats()
        launches = sum(v[0] for v in ks.values()) / (a.iters + 3)
        comm.set_config(hvd._lib.HVD_CFG_PROFILE, 1)
        for i in range(4):
            comm.allreduce_average(preps[i % len(preps)], fusion_threshold=thr)
        torch.cuda.synchronize()
        comm.kernel_stats()
        for i in range(8):
            comm.allreduce_average(preps[i % len(preps)], fusion_threshold=thr)
        kst = comm.kernel_stats()
        comm.set_config(hvd._lib.HVD_CFG_PROFILE, 0)
        dev_us = sum(v[1] for v in kst.values()) * 1e3 / 8
        row = {"config": cfg, "model": model, "dtype": dt, "fusion_threshold": thr, "tensors": len(counts),
               "device_us_per_allreduce": dev_us,
               "payload_bytes": payload, "us_per_allreduce": us, "busbw_GBps": bus(payload, us, n),
               "launches_per_call": launches}
        if n > 1:  # NCCL on the same tensors, one all_reduce per tensor (no fusion) and on one flat buffer
            flat = torch.cat([t.view(-1) for t in sets[0]])
            us_flat = timed(lambda i: dist.all_reduce(flat, group=ng), a.iters)
            row["nccl_flat_us"] = us_flat
            if thr == 0:
                us_each = timed(lambda i: [dist.all_reduce(t, group=ng) for t in sets[i % len(sets)]],
                                max(3, a.iters // 4))
                row["nccl_per_tensor_us"] = us_each
        res["rows"].append(row)
        if dist.get_rank() == 0:
            print(json.dumps(row), flush=True)

    if "C2" in only:
        model_row("C2", "resnet101", "f32", 64 * MIB)
    if "C3" in only:
        for dt in ("f32", "bf16"):
            model_row("C3", "inception_v3", dt, 64 * MIB)
            model_row("C3", "inception_v3", dt, 0)
    if "C4" in only:
        model_row("C4", "vgg16", "f32", 64 * MIB)
    if "C5" in only:
        for dt in ("f32", "bf16"):
            tdt = torch.float32 if dt == "f32" else torch.bfloat16
            esz = 4 if dt == "f32" else 2
            for lg in range(a.sweep_min_log2, a.sweep_max_log2 + 1):
                size = 1 << lg
                cnt = size // esz
                sets = sets_for([cnt], tdt, size)
                preps = [comm.prepare(st) for st in sets]
                iters = a.iters if size <= 256 * MIB else max(3, a.iters // 4)
                us = timed(lambda i: comm.allreduce_average(preps[i % len(preps)]), iters, nsets=len(preps))
                row = {"config": "C5", "dtype": dt, "bytes": size, "us": us, "busbw_GBps": bus(size, us, n),
                       "ll_max": comm.get_config(hvd._lib.HVD_CFG_LL_MAX_BYTES),
                       "ll128_max": comm.get_config(hvd._lib.HVD_CFG_LL128_MAX_BYTES)}
                if n > 1 and not a.no_nccl:
                    x = sets[0][0]
                    row["nccl_us"] = timed(lambda i: dist.all_reduce(x, group=ng), iters)
                    row["nccl_busbw_GBps"] = bus(size, row["nccl_us"], n)
                    row["nccl_env"] = os.environ.get("NCCL_ALGO", "default") + "/" + os.environ.get("NCCL_PROTO", "default")
                res["rows"].append(row)
                if dist.get_rank() == 0:
                    print(json.dumps(row), flush=True)
                del sets
    assert comm.poll_error() == 0
    if dist.get_rank() == 0:
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)
    dist.barrier()
    comm.finalize()


if __name__ == "__main__":
    main()

"""One 64 MiB fp32 gradient, allreduce-average at N GPUs: registered (the bench's zero-copy
path) against a plain tensor list (all-gather through the fusion buffer plus the final
local scatter), with HVD_CFG_FIN_LAG / CHANNELS / SLICE_BYTES variants, and each variant's
device timeline summary (busy time per phase, waits).  torchrun, one process per GPU;
rank 0 prints one JSON object and writes gpurun_out/nonreg_probe_n<N>.json."""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1802_05799_b200 as hvd  # noqa: E402
from paper_1802_05799_b200 import timeline  # noqa: E402


def tmax(x):
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("gloo")
    mib = int(os.environ.get("NR_MIB", "64"))
    comm = hvd.init(64 << 20)
    L = hvd._lib
    comm.set_config(L.HVD_CFG_TIMEOUT_MS, 60000)
    comm.set_config(L.HVD_CFG_LL128_MAX_BYTES, 0)
    x = torch.randn((mib << 20) // 4, device="cuda")
    reg = comm.register([x])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s = torch.cuda.current_stream()

    def timed(h, iters=40):
        for _ in range(5):
            comm.allreduce_average(h)
        torch.cuda.synchronize()
        dist.barrier()
        e0.record(s)
        for _ in range(iters):
            comm.allreduce_average(h)
        e1.record(s)
        torch.cuda.synchronize()
        return tmax(e0.elapsed_time(e1) / iters * 1e3)

    def tl_summary(h):
        comm.set_config(L.HVD_CFG_TIMELINE, 1024)
        comm.allreduce_average(h)
        torch.cuda.synchronize()
        dist.barrier()
        comm.allreduce_average(h)
        torch.cuda.synchronize()
        t = comm.timeline()
        comm.set_config(L.HVD_CFG_TIMELINE, 0)
        sm = timeline.summarize(t)
        sm["K"] = t["K"]
        return sm

    variants = [("registered", {}), ("plain", {})]
    for lag in (0, 2, 4, 64):
        variants.append((f"plain_fin_lag{lag}", {"FIN_LAG": lag}))
    for sb in (64, 32):
        variants.append((f"plain_slice{sb}k", {"SLICE_BYTES": sb << 10}))
        variants.append((f"registered_slice{sb}k", {"SLICE_BYTES": sb << 10}))
    variants.append(("plain_ch148", {"CHANNELS": 148}))
    variants.append(("registered_ch148", {"CHANNELS": 148}))
    defaults = {k: comm.get_config(getattr(L, "HVD_CFG_" + k)) for k in ("FIN_LAG", "SLICE_BYTES", "CHANNELS")}
    out = {"n": world, "mib": mib, "defaults": defaults, "runs": {}}
    for name, knobs in variants:
        for k, v in defaults.items():
            comm.set_config(getattr(L, "HVD_CFG_" + k), v)
        for k, v in knobs.items():
            comm.set_config(getattr(L, "HVD_CFG_" + k), v)
        h = reg if name.startswith("registered") else [x]
        us = timed(h)
        out["runs"][name] = {"us": us, "busbw_GBps": (mib << 20) / (us * 1e-6) / 1e9 * 2 * (world - 1) / world,
                             "timeline_rank0": tl_summary(h) if name in ("registered", "plain") else None}
        if rank == 0:
            print(name, round(us, 1), flush=True)
    if rank == 0:
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", f"nonreg_probe_n{world}.json"), "w") as f:
            json.dump(out, f, indent=1)
        print(json.dumps(out))
    dist.barrier()
    comm.finalize()


if __name__ == "__main__":
    main()

"""Capture a Horovod-style Timeline of one fused allreduce on every rank.

torchrun --nproc-per-node N tools/timeline_capture.py --mib 64 --out gpurun_out/timeline_n2.json
Writes a Chrome trace (chrome://tracing) merged over ranks and prints a per-rank summary.
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_05799_b200 as hvd  # noqa: E402
from paper_1802_05799_b200 import timeline  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=64)
    ap.add_argument("--out", default="gpurun_out/timeline.json")
    ap.add_argument("--channels", type=int, default=0)
    ap.add_argument("--slice-kib", type=int, default=0)
    ap.add_argument("--registered", action="store_true", help="registered tensor (the bench's path)")
    ap.add_argument("--config", action="append", default=[], metavar="KEY=VALUE", help="hvd_set_config")
    ap.add_argument("--summary-out", default="")
    a = ap.parse_args()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group("gloo")
    comm = hvd.init(fusion_bytes=max(64, a.mib) << 20)
    L = hvd._lib
    if a.channels:
        comm.set_config(L.HVD_CFG_CHANNELS, a.channels)
    if a.slice_kib:
        comm.set_config(L.HVD_CFG_SLICE_BYTES, a.slice_kib << 10)
    for kv in a.config:
        k, v = kv.split("=")
        comm.set_config(getattr(L, "HVD_CFG_" + k), int(v))
    comm.set_config(L.HVD_CFG_TIMELINE, 1024)
    x = torch.randn((a.mib << 20) // 4, device="cuda")
    h = comm.register([x]) if a.registered else [x]
    for _ in range(5):
        comm.allreduce_average(h)
    torch.cuda.synchronize()
    dist.barrier()
    comm.allreduce_average(h)
    torch.cuda.synchronize()
    tl = comm.timeline()
    allt = [None] * dist.get_world_size()
    dist.all_gather_object(allt, tl)
    if dist.get_rank() == 0:
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        timeline.write_chrome_trace(a.out, allt)
        summ = [timeline.summarize(t) for t in allt]
        print(json.dumps(summ, indent=1))
        with open(a.out.replace(".json", "_summary.json"), "w") as f:
            json.dump(summ, f, indent=1)
    dist.barrier()
    comm.finalize()


if __name__ == "__main__":
    main()

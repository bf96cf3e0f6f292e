"""hvd_allreduce_host (the bench's e2e path) at N GPUs: per-step time for chunk sizes and
protocol limits, and the H2D / D2H copy times alone, to find what slows it at N > 1.
torchrun, one process per GPU; rank 0 writes gpurun_out/e2e_probe_n<N>.json."""
import json
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1802_05799_b200 as hvd  # noqa: E402


def tmax(x):
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("gloo")
    comm = hvd.init(64 << 20)
    L = hvd._lib
    n = 16 << 20
    hin = torch.randn(n).pin_memory()
    hout = torch.empty(n).pin_memory()
    dev = torch.empty(n, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn, iters=10):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
        return tmax(e0.elapsed_time(e1) / iters)

    rows = {}
    rows["h2d_64MiB_ms"] = timed(lambda: dev.copy_(hin, non_blocking=True))
    rows["d2h_64MiB_ms"] = timed(lambda: hout.copy_(dev, non_blocking=True))
    rows["device_allreduce_64MiB_ms"] = timed(lambda: comm.allreduce_average([dev]))
    for ll128 in (1, 0):
        comm.set_config(L.HVD_CFG_LL128_MAX_BYTES, (16 << 20 if world == 2 else 32 << 20) if ll128 else 0)
        for chunk in (1 << 20, 2 << 20, 4 << 20, 8 << 20, 16 << 20, 32 << 20, 64 << 20):
            rows[f"e2e_ms_chunk{chunk >> 20}MiB_ll128{ll128}"] = timed(
                lambda: comm.allreduce_host(hin, hout, op="average", chunk_bytes=chunk))
    t0 = time.perf_counter()
    comm.allreduce_host(hin, hout, op="average")
    torch.cuda.synchronize()
    rows["e2e_host_wall_ms_one"] = (time.perf_counter() - t0) * 1e3
    if rank == 0:
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", f"e2e_probe_n{world}.json"), "w") as f:
            json.dump(rows, f, indent=1)
        print(json.dumps(rows))
    dist.barrier()
    comm.finalize()


if __name__ == "__main__":
    main()

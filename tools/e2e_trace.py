"""Job timeline of hvd_allreduce_host with small chunks (the e2e slow case): kernel spans
per chunk, per rank.  torchrun; writes gpurun_out/e2e_trace_n<N>_c<MiB>.json (the trace)."""
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1802_05799_b200 as hvd  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("gloo")
    chunk = int(os.environ.get("E2E_CHUNK_MIB", "4")) << 20
    path = os.path.join(ROOT, "gpurun_out", f"e2e_trace_n{world}_c{chunk >> 20}.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    comm = hvd.init(64 << 20)
    n = 16 << 20
    hin = torch.randn(n).pin_memory()
    hout = torch.empty(n).pin_memory()
    for _ in range(2):
        comm.allreduce_host(hin, hout, op="average", chunk_bytes=chunk)
    torch.cuda.synchronize()
    dist.barrier()
    comm.timeline_start(path)
    for _ in range(2):
        comm.allreduce_host(hin, hout, op="average", chunk_bytes=chunk)
    torch.cuda.synchronize()
    comm.timeline_stop()
    dist.barrier()
    comm.finalize()


if __name__ == "__main__":
    main()

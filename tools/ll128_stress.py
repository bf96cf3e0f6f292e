"""LL128 stress (torchrun, one process per GPU): many back-to-back LL128 allreduces of
random sizes, each compared bit for bit with the same call through the fused push
protocol (LL128 off).  A torn 128-byte line would show up as a mismatch.  Rank 0
prints one JSON line.  Self-consistency evidence for DESIGN.md's LL128 assumption; the
oracle parity of LL128 is in tests/test_gpu_virtual.py / test_gpu_multiprocess.py."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_05799_b200 as hvd  # noqa: E402


def main():
    calls = int(sys.argv[1]) if len(sys.argv) > 1 else 400
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    comm = hvd.init()
    L = hvd._lib
    g = torch.Generator(device="cuda").manual_seed(77 + rank)
    gen = torch.Generator().manual_seed(5)  # same sizes on every rank
    mismatches = 0
    total_bytes = 0
    for i in range(calls):
        n = int(torch.randint(70_000, 4_000_000, (1,), generator=gen))
        dt = torch.float32 if i % 2 == 0 else torch.bfloat16
        x = torch.randn(n, generator=g, device="cuda").to(dt)
        a, b = x.clone(), x.clone()
        comm.set_config(L.HVD_CFG_LL_MAX_BYTES, 0)
        comm.set_config(L.HVD_CFG_LL128_MAX_BYTES, 64 << 20)
        comm.allreduce_average([a])                      # LL128
        comm.set_config(L.HVD_CFG_LL128_MAX_BYTES, 0)
        comm.allreduce_average([b])                      # fused push
        torch.cuda.synchronize()
        mismatches += int((a.view(torch.int16 if dt == torch.bfloat16 else torch.int32) !=
                           b.view(torch.int16 if dt == torch.bfloat16 else torch.int32)).sum())
        total_bytes += n * x.element_size()
    assert comm.poll_error() == 0
    t = torch.tensor([mismatches], dtype=torch.int64)
    dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"calls": calls, "ranks": dist.get_world_size(), "bytes_reduced_per_rank": total_bytes,
                          "mismatched_elements": int(t.item())}), flush=True)
    dist.barrier()
    comm.finalize()


if __name__ == "__main__":
    main()

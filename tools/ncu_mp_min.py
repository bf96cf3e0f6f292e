"""ncu diagnostic for multi-process jobs (rank 0 under ncu, rank 1 plain): mode 3 = gloo
world 2 + torch kernels; 4 = hvd.init (+ HVD_NVLINK_CHECK=0 from the caller) + allreduce."""
import os
import sys

import torch
import torch.distributed as dist

mode = int(sys.argv[1])
rank = int(os.environ["RANK"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
x = torch.randn(1 << 22, device="cuda")
for _ in range(3):
    x.mul_(1.0)
torch.cuda.synchronize()
print("torch kernels done", flush=True)
if mode >= 4:
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1802_05799_b200 as hvd
    c = hvd.init(64 << 20)
    print("init done", flush=True)
    for _ in range(3):
        c.allreduce_average([x])
    torch.cuda.synchronize()
    print("allreduce done", flush=True)
    dist.barrier()
    c.finalize()
dist.barrier()
print("ok", mode, flush=True)
sys.stdout.flush()
os._exit(0)

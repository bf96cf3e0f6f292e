"""ncu diagnostic: does ncu intercept kernels of this process (mode 0: plain torch; 1: with a
gloo process group of world 1; 2: the library's virtual N=1 allreduce)."""
import os
import sys

import torch

mode = int(sys.argv[1])
if mode >= 1:
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29777")
    dist.init_process_group("gloo", rank=0, world_size=1)
x = torch.randn(1 << 20, device="cuda")
for _ in range(3):
    x.mul_(1.0)
if mode >= 2:
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1802_05799_b200 as hvd
    c = hvd.init_virtual(1, 0, 64 << 20)
    for _ in range(3):
        c.allreduce_average([[x]])
    c.finalize()
torch.cuda.synchronize()
print("ok", mode)

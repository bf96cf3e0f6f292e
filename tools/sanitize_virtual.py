"""Small virtual-rank workload for compute-sanitizer (memcheck / racecheck / synccheck).

  compute-sanitizer --tool memcheck python tools/sanitize_virtual.py
Covers: fused allreduce (fp32, bf16 wire), three-kernel path, pull protocol,
broadcast, allgather, registered tensors, on N = 3 virtual ranks, small sizes.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_05799_b200 as hvd  # noqa: E402

n = 3
L = hvd._lib
comm = hvd.init_virtual(n, 0, 1 << 20)
comm.set_config(L.HVD_CFG_CHANNELS, 4)
counts = [3, 1000, 70_001, 5]
ts = [[torch.randn(c, device="cuda") for c in counts] for _ in range(n)]
comm.allreduce_average(ts)
comm.allreduce(ts, op="average", wire="bf16")
comm.set_config(L.HVD_CFG_FUSED, 0)
comm.allreduce_average(ts)
comm.set_config(L.HVD_CFG_FUSED, 1)
comm.set_config(L.HVD_CFG_PROTOCOL, 0)
comm.allreduce_average(ts)
comm.set_config(L.HVD_CFG_PROTOCOL, 1)
comm.broadcast(ts, root=1)
ins = [torch.randn(4097, device="cuda") for _ in range(n)]
outs = [torch.empty(n * 4097, device="cuda") for _ in range(n)]
comm.allgather(ins, outs)
reg = comm.register(ts)
comm.allreduce_average(reg)
torch.cuda.synchronize()
assert comm.poll_error() == 0
comm.finalize()
print("sanitize workload ok")

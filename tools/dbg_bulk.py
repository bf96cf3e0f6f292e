import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.getcwd() + "/tests")
import torch, workloads, oracle
import paper_1802_05799_b200 as hvd
from hvd_testutil import to_torch, from_torch, assert_same
n = 2
c = hvd.init_virtual(n, 0, 64 << 20)
L = hvd._lib
c.set_config(L.HVD_CFG_TIMEOUT_MS, 2000)
c.set_config(L.HVD_CFG_PROTOCOL, 2)
c.set_config(L.HVD_CFG_LL_MAX_BYTES, 0)
c.set_config(L.HVD_CFG_LL128_MAX_BYTES, 0)
for counts in ([4096], [1000], [1 << 20], [1, 3, 64, 1000, 4097, 100_003, 7, 262_149, 0, 33]):
    xs = workloads.all_ranks(counts, "f32", n)
    ref, _, plan = oracle.allreduce(xs, ["f32"] * len(counts), "average", threshold=400_000)
    ts = [[to_torch(x, "f32") for x in xs[r]] for r in range(n)]
    c.allreduce(ts, op="average", fusion_threshold=400_000)
    torch.cuda.synchronize()
    print(counts[:4], "err", c.poll_error(), flush=True)
    if c.poll_error():
        break
    for r in range(n):
        for k in range(len(counts)):
            assert_same(from_torch(ts[r][k], "f32"), ref[r][k], "f32", f"r={r} k={k}")
    print("ok", flush=True)

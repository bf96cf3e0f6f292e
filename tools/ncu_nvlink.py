"""One rank of a real multi-GPU job running the bench step (one registered 64 MiB fp32
gradient, allreduce-average) for ncu NVLink counters (tools/ncu_nvlink.sh runs rank 0
under ncu, the others plain: ncu serialises profiled kernels, so only one rank is
profiled; its peers wait in the launch handshake).

Writes gpurun_out/nvlink/rank<r>.json: the launch count, the device traffic counters
(hvd_traffic: bytes this rank pushed to its successor) and the algorithmic bytes per
launch (2L - |c_{r+1}| - |c_{r+2}|) * esz of SURVEY §8(d) from the chunk bounds.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1802_05799_b200 as hvd
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    iters = int(os.environ.get("NVL_ITERS", "6"))
    protocol = int(os.environ.get("NVL_PROTOCOL", "1"))
    comm = hvd.init(64 << 20)
    comm.set_config(hvd._lib.HVD_CFG_TIMEOUT_MS, 120000)
    comm.set_config(hvd._lib.HVD_CFG_PROTOCOL, protocol)
    L = 16 << 20
    g = torch.randn(L, device="cuda")
    reg = comm.register([g])
    s0, n0 = comm.traffic()
    for _ in range(iters):
        comm.allreduce_average(reg)
    torch.cuda.synchronize()
    s1, n1 = comm.traffic()
    assert comm.poll_error() == 0
    b = hvd.chunk_bounds(L, world, hvd.HVD_FLOAT32)
    size = [int(b[c + 1] - b[c]) for c in range(world)]
    alg = (2 * L - size[(rank + 1) % world] - size[(rank + 2) % world]) * 4
    out = {"rank": rank, "world": world, "launches": iters, "protocol": protocol,
           "pushed_bytes_per_launch": (s1 - s0) / iters, "sends_per_launch": (n1 - n0) / iters,
           "algorithmic_bytes_per_launch": alg, "payload_bytes": L * 4}
    d = os.path.join(ROOT, "gpurun_out", "nvlink")
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, f"rank{rank}_n{world}_p{protocol}.json"), "w") as f:
        json.dump(out, f, indent=1)
    import torch.distributed as dist
    dist.barrier()
    comm.finalize()


if __name__ == "__main__":
    main()

"""N = 1 stream probe: the solo kernel (hvd_allreduce_average at N = 1) vs torch's own
elementwise kernels on the same cold-input pattern (64 MiB fp32, sets rotated over > 2 x L2).
Prints one JSON line per variant: us per call and GB/s of read+write bytes."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_05799_b200 as hvd  # noqa: E402

MIB = 1 << 20


def timeit(fn, nsets, iters=60, warm=8):
    for i in range(warm):
        fn(i % nsets)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        fn(i % nsets)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


def main():
    cnt = 16 * MIB
    S = cnt * 4
    nsets = 4
    xs = [torch.randn(cnt, device="cuda") for _ in range(nsets)]
    ys = [torch.empty(cnt, device="cuda") for _ in range(nsets)]
    comm = hvd.init(fusion_bytes=64 * MIB)
    regs = [comm.register([x]) for x in xs]
    rows = []
    us = timeit(lambda i: comm.allreduce_average(regs[i]), nsets)
    rows.append({"variant": "hvd solo", "us": us})
    comm.set_config(hvd._lib.HVD_CFG_PROFILE, 1)
    comm.kernel_stats()
    us = timeit(lambda i: comm.allreduce_average(regs[i]), nsets)
    ks = comm.kernel_stats()
    comm.set_config(hvd._lib.HVD_CFG_PROFILE, 0)
    rows.append({"variant": "hvd solo, HVD_CFG_PROFILE=1 (events around each launch)", "us": us,
                 "kernel_avg_us": ks["solo"][1] / ks["solo"][0] * 1e3})
    rows.append({"variant": "torch x.mul_(1.0)", "us": timeit(lambda i: xs[i].mul_(1.0), nsets)})
    rows.append({"variant": "torch y.copy_(x)", "us": timeit(lambda i: ys[i].copy_(xs[i]), nsets)})
    rows.append({"variant": "torch x.mul_(1.0) warm (1 set)", "us": timeit(lambda i: xs[0].mul_(1.0), 1)})
    big_x = torch.randn(256 * MIB, device="cuda")
    big_y = torch.empty_like(big_x)
    us = timeit(lambda i: big_y.copy_(big_x), 1, iters=10, warm=2)
    rows.append({"variant": "torch copy 1 GiB", "us": us, "bytes": 2 * big_x.numel() * 4})
    for r in rows:
        r["GBps"] = r.get("bytes", 2 * S) / (r["us"] * 1e-6) / 1e9
        print(json.dumps(r), flush=True)
    comm.finalize()


if __name__ == "__main__":
    main()

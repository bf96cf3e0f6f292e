"""Single-GPU workload for ncu: N virtual ranks, one fused allreduce-average per call.

  python tools/prof_virtual.py --n 2 --mib 64 --fused 1 --iters 3
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_05799_b200 as hvd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2)
    ap.add_argument("--mib", type=int, default=64)
    ap.add_argument("--fused", type=int, default=1)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--channels", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--slice-kib", type=int, default=0)
    ap.add_argument("--time", action="store_true")
    ap.add_argument("--model", default="")
    ap.add_argument("--dtype", default="f32")
    a = ap.parse_args()
    L = hvd._lib
    comm = hvd.init_virtual(a.n, 0, a.mib << 20)
    comm.set_config(L.HVD_CFG_FUSED, a.fused)
    if a.channels:
        comm.set_config(L.HVD_CFG_CHANNELS, a.channels)
    if a.threads:
        comm.set_config(L.HVD_CFG_THREADS, a.threads)
    if a.slice_kib:
        comm.set_config(L.HVD_CFG_SLICE_BYTES, a.slice_kib << 10)
    comm.set_config(L.HVD_CFG_PROFILE, 1)
    tdt = torch.float32 if a.dtype == "f32" else torch.bfloat16
    if a.model:
        import workloads
        counts = [c for _, c in workloads.gradient_set(a.model)]
    else:
        counts = [(a.mib << 20) // 4]
    ts = [[torch.randn(c, device="cuda").to(tdt) for c in counts] for _ in range(a.n)]
    for _ in range(a.iters):
        comm.allreduce_average(ts)
    torch.cuda.synchronize()
    st = comm.kernel_stats()
    if a.time:
        print({k: (v[0], round(v[1] / max(1, v[0]) * 1e3, 1)) for k, v in st.items() if v[0]})
    assert comm.poll_error() == 0
    comm.finalize()


if __name__ == "__main__":
    main()

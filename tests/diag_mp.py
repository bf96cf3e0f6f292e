"""Diagnose a multi-process case sequence (torchrun): run tests/test_gpu_multiprocess CASES
(optionally a subset) and report, per rank, which elements differ from the oracle."""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))  # (this script lives in tests/: it calls the oracle)
import oracle  # noqa: E402
import paper_1802_05799_b200 as hvd  # noqa: E402
import workloads  # noqa: E402
from hvd_testutil import from_torch, to_torch  # noqa: E402
from test_gpu_multiprocess import CASES  # noqa: E402


def diff(g, r):
    isz = g.dtype.itemsize
    return np.where((g.view(np.uint8).reshape(-1, isz) != r.view(np.uint8).reshape(-1, isz)).any(1))[0]


def ranges(idx):
    if len(idx) == 0:
        return []
    out, s, p = [], idx[0], idx[0]
    for i in idx[1:]:
        if i != p + 1:
            out.append((int(s), int(p) + 1))
            s = i
        p = i
    out.append((int(s), int(p) + 1))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="", help="comma list of case indices (default all)")
    ap.add_argument("--ll-max", type=int, default=-1)
    a = ap.parse_args()
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group("gloo")
    n = dist.get_world_size()
    comm = hvd.init()
    if a.ll_max >= 0:
        comm.set_config(hvd._lib.HVD_CFG_LL_MAX_BYTES, a.ll_max)
    sel = [int(x) for x in a.cases.split(",")] if a.cases else list(range(len(CASES)))
    for ci in sel:
        kind, counts, dtype, op, thr = CASES[ci]
        if kind == "tensors":
            kd = "normal" if dtype in ("f32", "bf16") else "int_uniform"
            ts = [to_torch(workloads.rank_tensor(c, dtype, rank, k, kd), dtype) for k, c in enumerate(counts)]
            comm.allreduce(ts, op=op, fusion_threshold=thr)
            torch.cuda.synchronize()
            xs = [[workloads.rank_tensor(c, dtype, r, k, kd) for k, c in enumerate(counts)] for r in range(n)]
            ref, _, _ = oracle.allreduce(xs, [dtype] * len(counts), op, threshold=thr)
            for k in range(len(counts)):
                g = from_torch(ts[k], dtype)
                bad = diff(g, ref[rank][k])
                print(f"rank {rank} case {ci} {kind} {counts} tensor {k}: {len(bad)} bad {ranges(bad)[:8]}", flush=True)
        elif kind == "registered":
            ts = [torch.empty(c, device="cuda") for c in counts]
            reg = comm.register(ts)
            for it in range(2):
                for k, c in enumerate(counts):
                    ts[k].copy_(to_torch(workloads.rank_tensor(c, "f32", rank, k, seed=700 + it), "f32"))
                comm.allreduce_average(reg, fusion_threshold=thr)
                torch.cuda.synchronize()
                xs = [[workloads.rank_tensor(c, "f32", r, k, seed=700 + it) for k, c in enumerate(counts)]
                      for r in range(n)]
                ref, _, plan = oracle.allreduce(xs, ["f32"] * len(counts), "average", threshold=thr)
                for k in range(len(counts)):
                    g = from_torch(ts[k], "f32")
                    bad = diff(g, ref[rank][k])
                    rr = ranges(bad)
                    print(f"rank {rank} case {ci} registered it {it} tensor {k}: {len(bad)} bad {rr[:12]}",
                          flush=True)
                    if len(bad):
                        i = bad[0]
                        own = xs[rank][k]
                        print(f"   first bad {i}: got {g[i]} want {ref[rank][k][i]} own {own[i]} "
                              f"succ {xs[(rank + 1) % n][k][i]} ptr {hex(ts[k].data_ptr())}", flush=True)
            comm.deregister(reg)
        elif kind == "negotiated":
            import random
            g = hvd.negotiator(comm, max_tensors=64)
            ts = [to_torch(workloads.rank_tensor(c, dtype, rank, k, "normal"), dtype) for k, c in enumerate(counts)]
            order = list(range(len(counts)))
            random.Random(1000 + rank).shuffle(order)
            for cyc in range(3):
                for tid in order[cyc::3]:
                    g.ready(tid, counts[tid], dtype)
                ids = comm.allreduce_negotiated(g, ts, op="average", fusion_threshold=thr)
                print(f"rank {rank} case {ci} cycle {cyc} ids {ids}", flush=True)
            torch.cuda.synchronize()
            g.close()
        elif kind == "host":
            x = workloads.rank_tensor(counts[0], dtype, rank, 5, "normal")
            hin = to_torch(x, dtype, device="cpu").pin_memory()
            hout = torch.empty_like(hin).pin_memory()
            comm.allreduce_host(hin, hout, op=op, chunk_bytes=thr)
            torch.cuda.synchronize()
            xs = [workloads.rank_tensor(counts[0], dtype, r, 5, "normal") for r in range(n)]
            ce = thr // oracle.ELEM_SIZE[dtype]
            bad = 0
            for off in range(0, counts[0], ce):
                ref, _, _ = oracle.allreduce([[xx[off:off + ce]] for xx in xs], [dtype], op)
                b = diff(from_torch(hout[off:off + ce], dtype), ref[rank][0])
                bad += len(b)
            print(f"rank {rank} case {ci} host: {bad} bad, err {comm.poll_error()}", flush=True)
        elif kind == "buffer":
            L = counts[0]
            x = workloads.rank_tensor(L, dtype, rank, 9, "normal" if dtype in ("f32", "bf16") else "int_uniform")
            tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "i32": torch.int32, "i64": torch.int64}[dtype]
            comm.fusion_buffer(0, tdt, L).copy_(to_torch(x, dtype))
            comm.allreduce_buffer(L, hvd._lib.__dict__["HVD_" + {"f32": "FLOAT32", "bf16": "BFLOAT16"}[dtype]], op)
            torch.cuda.synchronize()
            print(f"rank {rank} case {ci} buffer done", flush=True)
        elif kind == "bcast":
            xs = [workloads.rank_tensor(c, dtype, rank, k, "specials") for k, c in enumerate(counts)]
            ts = [to_torch(x, dtype) for x in xs]
            comm.broadcast(ts, root=op)
            torch.cuda.synchronize()
            print(f"rank {rank} case {ci} bcast done", flush=True)
        print(f"rank {rank} case {ci} err {comm.poll_error()}", flush=True)
    dist.barrier()
    comm.finalize()


if __name__ == "__main__":
    main()

"""Host <-> device copy bandwidth per rank, alone and all ranks at once (torchrun, one
process per GPU): what bounds the e2e path (hvd_allreduce_host) at N > 1.

Variants: pinned host memory from torch (pin_memory), and from cudaHostAlloc after the
process binds itself to the CPUs NVML reports as local to its GPU (first touch lands the
pages on that NUMA node).  64 MiB H2D and D2H, CUDA events, median of 10.
Writes gpurun_out/pcie/rank<r>.json.
"""
import json
import os
import subprocess
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def gpu_cpus(dev):
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(dev)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        cpus = [w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1]
        numa = None
        try:
            numa = pynvml.nvmlDeviceGetNumaNodeId(h)
        except Exception:
            pass
        return cpus, numa
    except Exception as e:
        return None, repr(e)


def bw(fn, nbytes, reps=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return nbytes / (ts[len(ts) // 2] / 1e3) / 1e9


def measure(host_in, host_out, dev_buf, nbytes, world, alone):
    res = {}
    rank = dist.get_rank()
    for what, fn in (("h2d", lambda: dev_buf.copy_(host_in, non_blocking=True)),
                     ("d2h", lambda: host_out.copy_(dev_buf, non_blocking=True)),
                     ("both", None)):
        if fn is None:
            s2 = torch.cuda.Stream()

            def fn():
                ev = torch.cuda.Event()
                ev.record()
                with torch.cuda.stream(s2):
                    s2.wait_event(ev)
                    host_out.copy_(dev_buf, non_blocking=True)
                dev_buf2.copy_(host_in, non_blocking=True)
                torch.cuda.current_stream().wait_stream(s2)
            dev_buf2 = torch.empty_like(dev_buf)
        if alone:
            vals = {}
            for r in range(world):
                dist.barrier()
                if r == rank:
                    vals = bw(fn, nbytes * (2 if what == "both" else 1))
                dist.barrier()
            res[what] = vals
        else:
            dist.barrier()
            res[what] = bw(fn, nbytes * (2 if what == "both" else 1))
    return res


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    nbytes = 64 << 20
    out = {"rank": rank, "world": world}
    cpus, numa = gpu_cpus(local)
    out["gpu_local_cpus"] = [cpus[0], cpus[-1], len(cpus)] if cpus else None
    out["gpu_numa_node"] = numa
    out["affinity_at_start"] = len(os.sched_getaffinity(0))
    dev = torch.empty(nbytes // 4, device="cuda")
    hin = torch.randn(nbytes // 4).pin_memory()
    hout = torch.empty(nbytes // 4).pin_memory()
    out["torch_pinned_alone"] = measure(hin, hout, dev, nbytes, world, True)
    out["torch_pinned_all"] = measure(hin, hout, dev, nbytes, world, False)
    if cpus:
        os.sched_setaffinity(0, cpus)
        hin2 = torch.empty(nbytes // 4).pin_memory()
        hin2.copy_(hin)
        hout2 = torch.empty(nbytes // 4).pin_memory()
        hout2.zero_()
        out["local_pinned_alone"] = measure(hin2, hout2, dev, nbytes, world, True)
        out["local_pinned_all"] = measure(hin2, hout2, dev, nbytes, world, False)
    if rank == 0:
        try:
            out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
            out["numactl"] = subprocess.run(["numactl", "-H"], capture_output=True, text=True).stdout
        except Exception as e:
            out["topo"] = repr(e)
    d = os.path.join(ROOT, "gpurun_out", "pcie")
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, f"rank{rank}_n{world}.json"), "w") as f:
        json.dump(out, f, indent=1)
    dist.barrier()


if __name__ == "__main__":
    sys.exit(main())

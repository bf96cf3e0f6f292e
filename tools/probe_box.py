"""One-off probe of a gpurun box: topology, P2P access, CUDA IPC across processes."""
import os, json, subprocess, sys
import torch
import torch.multiprocessing as mp

def child(q, h):
    t = h  # tensor shared via CUDA IPC by torch.multiprocessing
    torch.cuda.set_device(1)
    q.put(float(t.sum().item()))

def main():
    out = {}
    out["n"] = torch.cuda.device_count()
    out["name"] = torch.cuda.get_device_name(0)
    out["cpu_count"] = os.cpu_count()
    out["affinity"] = len(os.sched_getaffinity(0))
    try:
        out["cpu_model"] = [l for l in open("/proc/cpuinfo") if l.startswith("model name")][0].split(":")[1].strip()
    except Exception as e:
        out["cpu_model"] = str(e)
    if out["n"] >= 2:
        out["p2p01"] = torch.cuda.can_device_access_peer(0, 1)
        a = torch.ones(1 << 20, device="cuda:0")
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        p = ctx.Process(target=child, args=(q, a))
        p.start(); out["ipc_sum"] = q.get(timeout=120); p.join()
        # peer copy bandwidth
        x = torch.empty(1 << 28, dtype=torch.uint8, device="cuda:0")
        y = torch.empty(1 << 28, dtype=torch.uint8, device="cuda:1")
        for _ in range(3): y.copy_(x)
        torch.cuda.synchronize(0); torch.cuda.synchronize(1)
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); 
        for _ in range(10): y.copy_(x)
        e.record(); torch.cuda.synchronize(0); torch.cuda.synchronize(1)
        out["peer_copy_GBps"] = 10 * (1 << 28) / (s.elapsed_time(e) * 1e-3) / 1e9
    print(json.dumps(out))
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/probe.json", "w"))

if __name__ == "__main__":
    main()

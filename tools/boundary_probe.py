"""Where the time between back-to-back fused launches goes: the bench step (one registered
64 MiB fp32 gradient) at N GPUs, 40 calls back to back, with the job timeline (kernel begin
= first CTA start, end = last CTA end, %globaltimer) and the per-op device timeline of one
call (HVD_CFG_TIMELINE).  Per rank: period per call (CUDA events), kernel duration, gap from
one kernel's end to the next's begin, and the op span inside the kernel; kernel - span is
the launch handshake plus the final wait for the predecessor's last slices.
HVD_CFG_FUSED_PDL on and off.  torchrun; rank 0 writes gpurun_out/boundary_probe_n<N>.json."""
import json
import os
import statistics as st
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1802_05799_b200 as hvd  # noqa: E402
from paper_1802_05799_b200 import timeline  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("gloo")
    comm = hvd.init(64 << 20)
    L = hvd._lib
    comm.set_config(L.HVD_CFG_TIMEOUT_MS, 60000)
    x = torch.randn((64 << 20) // 4, device="cuda")
    reg = comm.register([x])
    out = {"n": world, "runs": {}}
    d = os.path.join(ROOT, "gpurun_out", "boundary")
    os.makedirs(d, exist_ok=True)
    for pdl in (0, 1):
        comm.set_config(L.HVD_CFG_FUSED_PDL, pdl)
        for _ in range(5):
            comm.allreduce_average(reg)
        torch.cuda.synchronize()
        dist.barrier()
        path = os.path.join(d, f"trace_n{world}_pdl{pdl}.json")
        comm.timeline_start(path)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        iters = 40
        for _ in range(iters):
            comm.allreduce_average(reg)
        e1.record()
        torch.cuda.synchronize()
        period = e0.elapsed_time(e1) / iters * 1e3
        comm.timeline_stop()
        dist.barrier()
        # one call with the per-op device timeline
        comm.set_config(L.HVD_CFG_TIMELINE, 1024)
        comm.allreduce_average(reg)
        torch.cuda.synchronize()
        span = timeline.summarize(comm.timeline())["span_us"]
        comm.set_config(L.HVD_CFG_TIMELINE, 0)
        ev = [e for e in timeline.load_trace(path) if e.get("cat") == "KERNEL" and e.get("ph") == "X"]
        per = []
        for pid in sorted({e["pid"] for e in ev}):
            ks = sorted((e for e in ev if e["pid"] == pid), key=lambda e: e["ts"])[5:]
            durs = [k["dur"] for k in ks]
            gaps = [b["ts"] - (a["ts"] + a["dur"]) for a, b in zip(ks, ks[1:])]
            per.append({"pid": pid, "kernels": len(ks), "dur_us_median": st.median(durs),
                        "gap_us_median": st.median(gaps) if gaps else None,
                        "gap_us_min": min(gaps) if gaps else None})
        info = {"period_us_rank": period, "op_span_us_rank": span}
        allinfo = [None] * world
        dist.all_gather_object(allinfo, info)
        out["runs"][f"pdl{pdl}"] = {"ranks": allinfo, "kernels": per}
        if rank == 0:
            print(f"pdl={pdl}", json.dumps(out["runs"][f"pdl{pdl}"]), flush=True)
    if rank == 0:
        with open(os.path.join(ROOT, "gpurun_out", f"boundary_probe_n{world}.json"), "w") as f:
            json.dump(out, f, indent=1)
    dist.barrier()
    comm.finalize()


if __name__ == "__main__":
    main()

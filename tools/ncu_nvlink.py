"""One rank of a real multi-GPU job running the bench step (one registered 64 MiB fp32
gradient, allreduce-average) for ncu NVLink counters (tools/ncu_nvlink.sh runs rank 0
under ncu, the others plain: ncu serialises profiled kernels, so only one rank is
profiled; its peers wait in the launch handshake).

Writes gpurun_out/nvlink/rank<r>.json: the launch count, the device traffic counters
(hvd_traffic: bytes this rank pushed to its successor), the algorithmic bytes per
launch (2L - |c_{r+1}| - |c_{r+2}|) * esz of SURVEY §8(d) from the chunk bounds, and the
GPU's NVLink byte counters read through NVML around the timed launches (data and raw
TX / RX over all links, KiB counters), so the link bytes are measured even without ncu.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


NVML_FIELDS = {"data_tx": 138, "data_rx": 139, "raw_tx": 140, "raw_rx": 141,
               "count_xmit": 202, "count_rcv": 204}


def nvml_nvlink(dev):
    """{name: counter summed over links} (None where the field is not supported)."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(dev)
    except Exception as e:  # pragma: no cover
        return {"error": repr(e)}
    out = {}
    for name, fid in NVML_FIELDS.items():
        tot, ok = 0, False
        for link in range(18):
            try:
                v = pynvml.nvmlDeviceGetFieldValues(h, [(fid, link)])[0]
                if v.nvmlReturn == 0:
                    tot += int(v.value.ullVal)
                    ok = True
            except Exception:
                pass
        out[name] = tot if ok else None
    return out


def main():
    import torch
    import paper_1802_05799_b200 as hvd
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    iters = int(os.environ.get("NVL_ITERS", "6"))
    protocol = int(os.environ.get("NVL_PROTOCOL", "1"))
    comm = hvd.init(64 << 20, pull_buffers=protocol == 0)
    comm.set_config(hvd._lib.HVD_CFG_TIMEOUT_MS, 120000)
    comm.set_config(hvd._lib.HVD_CFG_PROTOCOL, protocol)
    L = 16 << 20
    g = torch.randn(L, device="cuda")
    reg = comm.register([g])
    for _ in range(3):  # warm-up (plan upload, first-touch)
        comm.allreduce_average(reg)
    torch.cuda.synchronize()
    import torch.distributed as dist
    dist.barrier()
    s0, n0 = comm.traffic()
    v0 = nvml_nvlink(torch.cuda.current_device())
    for _ in range(iters):
        comm.allreduce_average(reg)
    torch.cuda.synchronize()
    v1 = nvml_nvlink(torch.cuda.current_device())
    s1, n1 = comm.traffic()
    assert comm.poll_error() == 0
    b = hvd.chunk_bounds(L, world, hvd.HVD_FLOAT32)
    size = [int(b[c + 1] - b[c]) for c in range(world)]
    alg = (2 * L - size[(rank + 1) % world] - size[(rank + 2) % world]) * 4
    out = {"rank": rank, "world": world, "launches": iters, "protocol": protocol,
           "pushed_bytes_per_launch": (s1 - s0) / iters, "sends_per_launch": (n1 - n0) / iters,
           "algorithmic_bytes_per_launch": alg, "payload_bytes": L * 4,
           "nvml_before": v0, "nvml_after": v1,
           "nvml_per_launch": {k: (v1[k] - v0[k]) / iters if isinstance(v0.get(k), int) and isinstance(v1.get(k), int)
                               else None for k in NVML_FIELDS},
           "nvml_units": "THROUGHPUT_* fields in KiB, COUNT_* in bytes (NVML field docs)"}
    d = os.path.join(ROOT, "gpurun_out", "nvlink")
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, f"rank{rank}_n{world}_p{protocol}.json"), "w") as f:
        json.dump(out, f, indent=1)
    dist.barrier()
    comm.finalize()
    sys.stdout.flush()
    os._exit(0)  # no interpreter teardown under ncu


if __name__ == "__main__":
    main()

"""Which NVLink byte counters this driver exposes: NVML field values per link and
aggregate (return codes), and nvidia-smi's nvlink throughput counters.  Diagnostic."""
import json
import os
import subprocess
import sys


def main():
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    out = {"driver": pynvml.nvmlSystemGetDriverVersion()}
    states = {}
    for link in range(18):
        try:
            states[link] = pynvml.nvmlDeviceGetNvLinkState(h, link)
        except Exception as e:
            states[link] = repr(e)
    out["link_state"] = states
    fields = {}
    for fid in (138, 139, 140, 141, 202, 204, 91):
        for scope in (0, 1, 0xFFFFFFFF):
            try:
                v = pynvml.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
                fields[f"{fid}/{scope}"] = [v.nvmlReturn, int(v.value.ullVal)]
            except Exception as e:
                fields[f"{fid}/{scope}"] = repr(e)
        try:
            v = pynvml.nvmlDeviceGetFieldValues(h, [fid])[0]
            fields[f"{fid}/plain"] = [v.nvmlReturn, int(v.value.ullVal)]
        except Exception as e:
            fields[f"{fid}/plain"] = repr(e)
    out["fields"] = fields
    for args in (["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"], ["nvidia-smi", "nvlink", "-s", "-i", "0"],
                 ["nvidia-smi", "nvlink", "-h"]):
        try:
            r = subprocess.run(args, capture_output=True, text=True, timeout=30)
            out[" ".join(args)] = (r.stdout + r.stderr)[-3000:]
        except Exception as e:
            out[" ".join(args)] = repr(e)
    d = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", "nvlink")
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "nvml_probe.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    sys.exit(main())

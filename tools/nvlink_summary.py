"""Summarise the ncu range captures of tools/r02/c13_nvlink_counters.sh (gpurun_out/nvlink/range_n*_p*_*.csv
+ the matching oneproc_*.json) into profiles/r02_nvlink_counters.json, per launch:
NVLink TX/RX user and protocol bytes on device 0 (rank 0), DRAM bytes, and the ratio of
user bytes to the algorithmic (2L - |c_{r+1}| - |c_{r+2}|) * esz of SURVEY §8(d)."""
import csv
import glob
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
D = os.path.join(ROOT, "gpurun_out", "nvlink")


def read_csv(p):
    with open(p) as f:
        lines = [ln for ln in f if not ln.startswith("==")]
    rows = list(csv.reader(lines))
    if not rows:
        return {}
    h = rows[0]
    out = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        try:
            out[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        except (KeyError, ValueError):
            pass
    return out


def main():
    res = {}
    for p in sorted(glob.glob(os.path.join(D, "range_n*_p*_*.csv"))):
        m = re.search(r"range_n(\d+)_p(\d+)_(\d+)\.csv", p)
        n, proto, mib = int(m.group(1)), int(m.group(2)), int(m.group(3))
        met = read_csv(p)
        js = os.path.join(D, f"oneproc_n{n}_p{proto}_{mib}MiB_ncu.json")
        plain = os.path.join(D, f"oneproc_n{n}_p{proto}_{mib}MiB.json")
        if not met or not os.path.exists(js):
            continue
        info = json.load(open(js))
        k = info["iters"]
        alg = info["per_rank"][0]["algorithmic_nvlink_bytes_per_launch"]
        e = {"n": n, "protocol": proto, "payload_MiB": mib, "launches_in_range": k,
             "kernels_rank0": info["kernels"]}
        for name in ("nvltx__bytes.sum", "nvltx__bytes_data_user.sum", "nvltx__bytes_data_protocol.sum",
                     "nvlrx__bytes.sum", "nvlrx__bytes_data_user.sum", "nvlrx__bytes_data_protocol.sum",
                     "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
            if name in met:
                e[name.replace(".sum", "") + "_per_launch"] = met[name] / k
        e["algorithmic_nvlink_bytes_per_launch"] = alg
        if "nvltx__bytes_data_user_per_launch" in e:
            e["tx_user_over_algorithmic"] = e["nvltx__bytes_data_user_per_launch"] / alg
            e["tx_protocol_over_user"] = e["nvltx__bytes_data_protocol_per_launch"] / e["nvltx__bytes_data_user_per_launch"]
        if os.path.exists(plain):
            pi = json.load(open(plain))
            e["plain_us_per_launch"] = pi["us_per_launch"]
            e["plain_busbw_GBps"] = pi["busbw_GBps"]
            e["plain_kernels_rank0"] = pi["kernels"]
            e["wire_GBps_tx_rank0"] = e.get("nvltx__bytes_per_launch", 0) / (pi["us_per_launch"] * 1e-6) / 1e9
        res[f"n{n}_p{proto}_{mib}MiB"] = e
    out = {"what": "ncu application-range replay of 10 back-to-back launches of the bench step (one "
                   "registered gradient, allreduce-average), counters of device 0 (rank 0); one process "
                   "drives all N GPUs (tools/nvlink_1proc.py: ncu cannot profile while another process "
                   "uses the GPUs on this pool, and kernel replay would serialise the ranks' launches). "
                   "Range timings run slower under ncu; plain_* are the same launches without ncu. "
                   "protocol 1 = SM-store push (fused_allreduce_kernel), 2 = TMA bulk push; "
                   "16 MiB runs the LL128 kernel.", "runs": res}
    with open(os.path.join(ROOT, "profiles", "r02_nvlink_counters.json"), "w") as f:
        json.dump(out, f, indent=1)
    for k, v in res.items():
        print(k, {a: (round(b, 4) if isinstance(b, float) else b) for a, b in v.items()
                  if a in ("tx_user_over_algorithmic", "tx_protocol_over_user", "plain_busbw_GBps",
                           "wire_GBps_tx_rank0", "plain_kernels_rank0")})


if __name__ == "__main__":
    main()

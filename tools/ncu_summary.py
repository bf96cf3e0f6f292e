"""Summarise an ncu --set full report (one kernel) into a small JSON for profiles/.

  python tools/ncu_summary.py gpurun_out/x.ncu-rep > profiles/r01_ncu_x.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Kernel Name", "Block Size", "Grid Size", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__time_duration.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__occupancy_limit_registers", "sm__cycles_active.avg", "gpc__cycles_elapsed.max"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], check=True, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for k in KEYS:
        if k in head:
            i = head.index(k)
            d[k] = (vals[i] + " " + units[i]).strip()
    stalls = []
    for i, k in enumerate(head):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                stalls.append((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(vals[i].replace(",", ""))))
            except ValueError:
                pass
    d["top_stall_reasons_samples"] = sorted(stalls, key=lambda x: -x[1])[:6]
    try:
        rd = float(vals[head.index("dram__bytes_read.sum")].replace(",", ""))
        wr = float(vals[head.index("dram__bytes_write.sum")].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        d["dram_bytes_total"] = rd * scale.get(units[head.index("dram__bytes_read.sum")], 1) + \
            wr * scale.get(units[head.index("dram__bytes_write.sum")], 1)
    except (ValueError, IndexError):
        pass
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])

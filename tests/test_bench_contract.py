"""bench.py's reference arm runs on CPU: check its JSON line against the driver contract
(the GPU arm's line is produced on the B200 box; profiles/r01_bench_*.json)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run("--impl", "reference", "--gpus", "2", "--steps", "3", "--warmup", "3")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["higher_is_better"] is True and d["config"]["workload"] == "fp32_64MiB"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    # host metadata next to the oracle timing
    assert cb["host_cpus"] >= 1 and cb["sched_getaffinity"] >= 1 and cb["threads_used"] == 1
    assert "cpu_model" in cb


def test_roofline_traffic_and_nvlink_counters_per_n():
    """bench.py's roofline reads the committed ncu summary per rank count: DRAM traffic of the
    solo kernel (N = 1) and of the fused kernel at N = 2 / 4, and the NVLink counters whose
    user bytes equal the algorithmic (2L - |c_{r+1}| - |c_{r+2}|) * esz within 0.1 %."""
    sys.path.insert(0, ROOT)
    import importlib
    bench = importlib.import_module("bench")
    assert bench._ncu_traffic("solo_kernel", 1) > 0
    for n in (2, 4):
        assert bench._ncu_traffic("fused_allreduce_kernel", n) > 0
        nv = bench._ncu_profile("fused_allreduce_kernel", n, "nvlink")
        assert abs(nv["nvltx_user_bytes"] / nv["algorithmic_bytes"] - 1) < 1e-3
        assert nv["nvlrx_user_bytes"] == nv["nvltx_user_bytes"]
        assert 0 < nv["protocol_over_user"] < 0.3


def test_committed_gpu_lines_follow_the_contract():
    """The GPU lines committed under profiles/ carry every key the driver reads."""
    for n, rnd in ((1, "r01"), (2, "r01"), (4, "r01"), (1, "r02"), (2, "r02"), (4, "r02")):
        p = os.path.join(ROOT, "profiles", f"{rnd}_bench_n{n}.json")
        if not os.path.exists(p):
            continue
        d = json.load(open(p))
        assert d["n_gpus"] == n and d["warmup"] >= 3 and d["gpu_launches"] > 0
        r = d["roofline"]
        for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
            assert k in r, k
        assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
        for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
            assert k in d["e2e"], k
        assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
        for k in ("sm_mhz", "sm_max_mhz", "reasons"):
            assert k in d["clocks"], k
        if n == 1:
            assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1

#!/usr/bin/env python
"""Benchmark of the fused ring allreduce (Horovod, arXiv 1802.05799) on B200.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W`` prints ONE
JSON line on rank 0.  For N > 1 it is launched by torchrun, one process per
GPU.  A "step" is one pass of the whole hot path — plan -> pack (x 1/N) ->
ring reduce-scatter + all-gather -> unpack — over one synthetic gradient set,
through the C ABI ``hvd_allreduce_average``.

Metric (BASELINE.json): fused ring-allreduce bus GB/s of a 64 MB fp32 gradient
buffer.  busBW = payload_bytes / t * 2(N-1)/N (nccl-tests convention; the
per-rank ring traffic of P:L197-204).  At N = 1 the ring has no iterations
(factor 0), so ``value`` is the algorithmic bandwidth payload_bytes / t of the
N = 1 path (pack/scale + unpack) and ``value_kind`` says so.

Timed region: K steps between barriers, CUDA events on the stream, max over
ranks, no per-launch events; inputs are registered gradient tensors rotated
over > 2 x L2.  ``roofline``: the dominant kernel (here the only kernel of a
step) with its algorithmic bytes per launch over its average launch duration
in the timed region; a second, profiled pass (events around every launch)
gives ``achieved_profiled`` and ``share_of_step``.  ``e2e``: the same metric
through ``comm.allreduce_host`` with pinned host gradients in and the averaged
result out (H2D / ring / D2H pipelined in 8 MiB chunks).  ``cpu_baseline``:
the oracle on a bounded sample, rank 0, N = 1 only.

``--impl reference`` times the CPU oracle (``oracle/``) — the only reference
this tier has — on the same workload, on rank 0 only: W warm-up + K steps of a
bounded per-step sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MIB = 1 << 20
METRIC = "fused ring-allreduce bus GB/s (64 MB fp32) at 2/4/8 B200 vs 900 GB/s NVLink"
NVLINK_NOMINAL_GBPS = 900.0
NVLINK_MEASURED_GBPS = 770.0  # B200_PROFILING.md: measured peer copy per direction per GPU
L2_BYTES = 126 * MIB


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def _workload_counts(name):
    import workloads
    if name == "fp32_64MiB":
        return [16 * MIB], "f32"           # one 64 MiB fp32 gradient = one full fusion buffer
    model, dt = name.rsplit("_", 1) if name.endswith(("_f32", "_bf16")) else (name, "f32")
    return [c for _, c in workloads.gradient_set(model)], dt


def _bus_factor(n):
    return 2.0 * (n - 1) / n if n > 1 else 0.0


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, devices):
        self.devices = devices
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()

    def summary(self, t0=None, t1=None):
        """Median SM clock and active throttle reasons over samples taken in [t0, t1] (epoch s)."""
        import datetime
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (getattr(self, "out", "") or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9 or not f[1].isdigit() or int(f[1]) not in self.devices:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                ts = None
            if t0 is not None and ts is not None and not (t0 - 0.15 <= ts <= t1 + 0.15):
                continue
            try:
                sm.append(float(f[2]))
                mx.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "window": "pre-load + timed region"}


# ---------------------------------------------------------------- distributed plumbing
def _dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", os.environ.get("RANK", "0")))


def _max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _barrier(world):
    import torch
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch

    import paper_1802_05799_b200 as hvd
    rank, world, local = _dist_env()
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    clk = ClockSampler({local} if world == 1 else set(range(world)))
    clk.__enter__()  # nvidia-smi needs ~1 s to start sampling: start it first
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    comm = hvd.init(fusion_bytes=64 * MIB, device=local, pull_buffers="PROTOCOL=0" in args.config)
    for kv in args.config:
        k, v = kv.split("=")
        comm.set_config(getattr(hvd._lib, "HVD_CFG_" + k), int(v))
    counts, dt = _workload_counts(args.workload)
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16}[dt]
    esz = 4 if dt == "f32" else 2
    payload = sum(counts) * esz
    # inputs larger than L2: rotate over enough gradient sets that the set a step
    # reads was evicted by the others (>= 2 x L2 of distinct gradient bytes)
    nsets = args.sets if args.sets else max(2, -(-2 * L2_BYTES // payload))
    g = torch.Generator(device="cuda").manual_seed(180205799 + rank)
    sets = [[torch.randn(c, generator=g, device="cuda", dtype=torch.float32).to(tdt) for c in counts]
            for _ in range(nsets)]
    L = hvd._lib
    # the timed region runs without per-launch events (they cost ~5 us of device time per
    # launch at N = 1); kernel durations come from a second, profiled pass below
    comm.set_config(L.HVD_CFG_PROFILE, 0)
    # the gradient tensors of a training loop persist across steps: register them once
    # (zero-copy both ways: the all-gather writes final values into the successor's tensors)
    handles = [comm.register(st) for st in sets] if args.registered else [comm.prepare(st) for st in sets]

    def step(i):
        comm.allreduce_average(handles[i % nsets])

    _barrier(world)
    w0 = time.perf_counter()
    for i in range(args.warmup):
        step(i)
    _barrier(world)
    # every rank must make the same number of collective calls: the pre-load
    # count is derived from a calibration run (the warm-up includes first-call
    # costs such as plan uploads) and agreed on (max over ranks)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    ncal = 50
    for i in range(ncal):
        step(i)
    torch.cuda.synchronize()
    per_step = (time.perf_counter() - w0) / ncal
    n_load = int(_max_over_ranks(min(200000.0, args.clock_window / max(per_step, 1e-6)), world))
    comm.kernel_stats()  # reset counters
    t_load0 = time.time()
    if True:
        # keep the GPU busy ~clock_window s so the sampler sees clocks under load, then time K steps
        for i in range(n_load):
            step(i)
            if i % 64 == 63:
                torch.cuda.synchronize()
        _barrier(world)
        comm.kernel_stats()
        _barrier(world)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for i in range(args.steps):
            step(i)
        s1.record()
        _barrier(world)
    t_load1 = time.time()
    clk.__exit__(None, None, None)
    ms_local = s0.elapsed_time(s1)
    ks_timed = comm.kernel_stats()  # launch counts of the timed region
    # profiled pass: the same K steps with CUDA events around every launch on its stream
    comm.set_config(L.HVD_CFG_PROFILE, 1)
    comm.kernel_stats()
    _barrier(world)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record()
    for i in range(args.steps):
        step(i)
    p1.record()
    _barrier(world)
    ks = comm.kernel_stats()
    comm.set_config(L.HVD_CFG_PROFILE, 0)
    ms_prof_local = p0.elapsed_time(p1)
    ms = _max_over_ranks(ms_local, world)
    t = ms / 1e3 / args.steps
    n = world
    algbw = payload / t / 1e9
    value = algbw * _bus_factor(n) if n > 1 else algbw

    # ---- roofline of the dominant kernel (device time of each launch, CUDA events on its stream)
    peaks = _peaks()
    kt = {k: (v[0], v[1]) for k, v in ks.items() if v[0]}
    dom = max(kt, key=lambda k: kt[k][1])
    launches, dev_ms = kt[dom]
    avg_s_prof = dev_ms / 1e3 / launches  # per-launch CUDA events (profiled pass)
    # When the dominant kernel is the only kernel of the step, its average launch duration
    # is measured over the timed region itself: the region's CUDA events (max over ranks)
    # / its launches, with no per-launch events adding device time
    timed_launches = {k: v[0] for k, v in ks_timed.items() if v[0]}
    only_dom = set(timed_launches) == {dom}
    avg_s = (ms / 1e3 / timed_launches[dom]) if only_dom else avg_s_prof
    esz_of = {"f32": 4, "bf16": 2}
    fplan = hvd.plan(counts, [dt] * len(counts))
    if dom in ("ring", "fused") and n > 1:
        # NVLink bytes this rank pushes per step: sum over fusion buffers of
        # (2L - |c_{r+1}| - |c_{r+2}|) * esz  (~ 2(N-1)/N * S)
        step_bytes = 0
        for bdt, Lb, _ in fplan:
            cb = hvd.chunk_bounds(Lb, n, bdt)
            sz = [cb[i + 1] - cb[i] for i in range(n)]
            step_bytes += (2 * Lb - sz[(rank + 1) % n] - sz[(rank + 2) % n]) * esz_of[bdt]
        per_launch = step_bytes * args.steps / launches
        roof = {"kernel": f"{dom}_allreduce_kernel", "bound": "nvlink", "unit": "GB/s",
                "achieved": per_launch / avg_s / 1e9, "peak": NVLINK_MEASURED_GBPS,
                "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s per direction (no NVLink figure in "
                               "MEASURED_PEAKS.json); nominal 900",
                "algorithmic_bytes_per_launch": per_launch}
        roof["frac"] = roof["achieved"] / roof["peak"]
        roof["frac_of_nominal_900"] = roof["achieved"] / NVLINK_NOMINAL_GBPS
    else:
        # HBM: fused at N=1 reads the members and writes them back; pack reads the
        # members + writes the buffer; unpack reads the buffer + writes the members
        if dom in ("fused", "solo"):
            step_bytes = 2 * payload
        else:
            step_bytes = payload + sum(Lb * esz_of[bdt] for bdt, Lb, _ in fplan)
        per_launch = step_bytes * args.steps / launches
        roof = {"kernel": f"{dom}_kernel", "bound": "hbm", "unit": "GB/s",
                "achieved": per_launch / avg_s / 1e9, "peak": peaks.get("hbm_gbs", 6650.0),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650",
                "algorithmic_bytes_per_launch": per_launch}
        roof["frac"] = roof["achieved"] / roof["peak"]
    roof["achieved_profiled"] = roof["achieved"] * avg_s / avg_s_prof
    roof["frac_profiled"] = roof["achieved_profiled"] / roof["peak"]
    # the committed ncu captures are of the default workload (one 64 MiB fp32 gradient)
    cap = args.workload == "fp32_64MiB"
    roof["traffic"] = _ncu_traffic(roof["kernel"], n) if cap else None
    if n > 1:
        nvc = _ncu_profile(roof["kernel"], n, "nvlink") if cap else None
        roof["nvlink_counters"] = nvc
        if nvc and roof["bound"] == "nvlink":
            # wire bytes on the link per launch = user (= algorithmic) bytes x (1 + the link's
            # measured protocol share): against the 900 GB/s raw per-direction NVLink rate
            wire = roof["achieved"] * nvc["user_over_algorithmic"] * (1 + nvc["protocol_over_user"])
            roof["wire_GBps"] = wire
            roof["frac_of_raw_link_900"] = wire / NVLINK_NOMINAL_GBPS
    roof["share_of_step"] = dev_ms / ms_prof_local if ms_prof_local else None
    roof["timing"] = (("achieved: the dominant kernel is the only kernel of the step, so its average launch "
                       "duration = the timed region's CUDA events (max over ranks) / its launches. " if only_dom else
                       "achieved: per-launch CUDA events of the profiled pass. ") +
                      "achieved_profiled / share_of_step: CUDA events around each launch on its stream in a second "
                      "pass of the same K steps (those events add ~3-5 us of device time per launch, so the timed "
                      "region runs without them)")
    roof["profiled_ms_per_step"] = ms_prof_local / args.steps
    kernels = {k: {"launches_per_step": v[0] / args.steps, "avg_us": v[1] / v[0] * 1e3} for k, v in kt.items()}
    gpu_launches = int(sum(v[0] for v in ks_timed.values()))

    # ---- headline ring only: hvd_allreduce_buffer on one 64 MiB fp32 buffer (no pack/unpack)
    ring_only = None
    if n > 1:
        cnt = 16 * MIB
        for _ in range(args.warmup):
            comm.allreduce_buffer(cnt, L.HVD_FLOAT32, "sum")
        comm.kernel_stats()
        _barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            comm.allreduce_buffer(cnt, L.HVD_FLOAT32, "sum")
        e1.record()
        _barrier(world)
        rms = _max_over_ranks(e0.elapsed_time(e1), world) / args.steps
        comm.kernel_stats()
        ring_only = {"bytes": cnt * 4, "us": rms * 1e3, "busbw_GBps": cnt * 4 / (rms / 1e3) / 1e9 * _bus_factor(n)}

    # ---- e2e: through the public API with HOST buffers: hvd_allreduce_host takes pinned host
    # gradients (one flat buffer, as a host-staged training loop holds them) and returns the
    # averaged result in host memory; chunked H2D -> ring -> D2H, pipelined
    host_in = torch.cat([t.view(-1) for t in sets[0]]).cpu().pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()
    e2e_steps = max(3, min(args.steps, 20))

    def e2e_step():
        comm.allreduce_host(host_in, host_out, op="average")

    for _ in range(2):
        e2e_step()
    _barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(e2e_steps):
        e2e_step()
    e1.record()
    _barrier(world)
    ems = _max_over_ranks(e0.elapsed_time(e1), world) / e2e_steps
    e_alg = payload / (ems / 1e3) / 1e9
    e2e = {"value": e_alg * _bus_factor(n) if n > 1 else e_alg, "unit": "GB/s", "h2d_bytes_per_step": payload,
           "d2h_bytes_per_step": payload, "ms_per_step": ems,
           "api": "comm.allreduce_host (hvd_allreduce_host): pinned host in/out, 8 MiB chunks, "
                  "H2D / ring / D2H overlapped"}
    assert comm.poll_error() == 0, hvd._lib.strerror(comm.poll_error())

    cpu = None
    if rank == 0 and n == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, counts, dt, n)

    clocks = clk.summary(t_load0, t_load1)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": n, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": dt, "data": "synthetic",
            "value_kind": "busBW = payload/t * 2(N-1)/N" if n > 1 else
                          "algBW = payload/t (N=1: the ring has no iterations, bus factor 0)",
            "config": {"workload": args.workload, "payload_bytes": payload, "tensors": len(counts),
                       "tensors_registered": bool(args.registered),
                       "fusion_bytes": 64 * MIB, "op": "average",
                       "l2": f"inputs rotate over {nsets} gradient sets ({nsets * payload / MIB:.0f} MiB "
                             + ("> 2 x L2: every step reads cold inputs)" if nsets * payload > 2 * L2_BYTES
                                else "<= 2 x L2: WARM inputs, not a contract measurement)"),
                       "parallelism": f"dp{n}", "ranks": "one process per GPU, CUDA-IPC ring",
                       **({"knobs": args.config} if args.config else {})},
            "roofline": roof, "kernels": kernels, "ring_only_64MiB": ring_only, "e2e": e2e,
            "gpu_launches": gpu_launches, "cpu_baseline": cpu, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    comm.finalize()


def _ncu_profile(kernel, n, key="dram"):
    """Per-launch counters of `kernel` at N ranks from the committed ncu summary
    (profiles/ncu_traffic.json): key "dram" -> dram__bytes_read + write (the roofline's
    `traffic`), key "nvlink" -> {nvltx user / protocol bytes, nvlrx user bytes}."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None
    v = d.get(kernel) if key == "dram" else d.get("nvlink", {}).get(kernel)
    if isinstance(v, dict):
        v = v.get(str(n))
    return v


def _ncu_traffic(kernel, n=1):
    return _ncu_profile(kernel, n, "dram")


# ---------------------------------------------------------------- CPU oracle (baseline / reference arm)
def _oracle_inputs(counts, dt, n, max_elems):
    """Seeded inputs of a bounded sample of the workload: the first tensors up to max_elems."""
    import workloads
    sample, tot = [], 0
    for c in counts:
        if tot >= max_elems:
            break
        take = min(c, max_elems - tot)
        sample.append(take)
        tot += take
    return sample, workloads.all_ranks(sample, dt, n)


def cpu_baseline(args, counts, dt, n, budget_s=10.0):
    import oracle
    esz = 4 if dt == "f32" else 2
    sample, xs = _oracle_inputs(counts, dt, n, 16 * MIB)
    payload = sum(sample) * esz
    dts = [dt] * len(sample)
    reps, t0 = 0, time.perf_counter()
    while True:
        oracle.allreduce(xs, dts, "average")
        reps += 1
        if time.perf_counter() - t0 > budget_s:
            break
    t = (time.perf_counter() - t0) / reps
    alg = payload / t / 1e9
    # C1: 1,048,576 fp32 x 4 simulated ranks, median of 5, seconds
    x4 = _oracle_inputs([1 << 20], "f32", 4, 1 << 20)[1]
    c1 = []
    for _ in range(5):
        s = time.perf_counter()
        oracle.allreduce(x4, ["f32"], "average")
        c1.append(time.perf_counter() - s)
    return {"value": alg * _bus_factor(n) if n > 1 else alg, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": f"oracle.allreduce of {len(sample)} tensor(s), {payload / MIB:.0f} MiB {dt} per rank, "
                      f"{n} simulated rank(s), {reps} reps in {reps * t:.1f} s (numpy, single thread)",
            "c1_seconds_median5": statistics.median(c1), **_host_info()}


def _host_info():
    """Host metadata BASELINE.md §4 asks for next to the oracle timing."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        aff = sorted(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        aff = None
    return {"host_cpus": os.cpu_count(), "sched_getaffinity": len(aff) if aff is not None else None,
            "cpu_model": model, "threads_used": 1,
            "omp_num_threads": os.environ.get("OMP_NUM_THREADS")}


def run_reference(args, budget_s=120.0):
    """The reference arm: the CPU oracle as it stands, on rank 0, W warm-up + K timed steps;
    each step is a bounded sample of the workload, sized so the whole run stays within
    ~budget_s (calibrated on a 1 Mi-element sample)."""
    rank, world, _ = _dist_env()
    if rank != 0:
        return
    import oracle
    counts, dt = _workload_counts(args.workload)
    n = args.gpus
    esz = 4 if dt == "f32" else 2
    small, xs_small = _oracle_inputs(counts, dt, n, 1 * MIB)
    t0 = time.perf_counter()
    oracle.allreduce(xs_small, [dt] * len(small), "average")
    per_elem = (time.perf_counter() - t0) / max(1, sum(small))
    per_step = budget_s / (args.steps + args.warmup)
    cap = int(min(16 * MIB, max(64 * 1024, per_step / max(per_elem, 1e-12))))
    sample, xs = _oracle_inputs(counts, dt, n, cap)
    payload = sum(sample) * esz
    dts = [dt] * len(sample)
    for _ in range(args.warmup):
        oracle.allreduce(xs, dts, "average")
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.allreduce(xs, dts, "average")
    t = (time.perf_counter() - t0) / args.steps
    alg = payload / t / 1e9
    value = alg * _bus_factor(n) if n > 1 else alg
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": n,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": dt, "data": "synthetic",
            "config": {"workload": args.workload, "payload_bytes": payload, "simulated_ranks": n},
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "sample": f"{len(sample)} tensor(s), {payload / MIB:.2f} MiB per rank of the "
                                       f"workload, {n} simulated rank(s), per step; numpy single thread",
                             **_host_info()},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="fp32_64MiB",
                    help="fp32_64MiB | resnet101 | inception_v3[_bf16] | vgg16")
    ap.add_argument("--clock-window", type=float, default=1.5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--registered", type=int, default=1, help="1: registered gradient tensors (zero-copy)")
    ap.add_argument("--sets", type=int, default=0, help="input sets to rotate (0: enough to exceed 2 x L2)")
    ap.add_argument("--config", action="append", default=[], metavar="KEY=VALUE",
                    help="hvd_set_config before timing, e.g. CHANNELS=64 (repeatable)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

#!/bin/bash
# Profiling pass for one round (run under gpurun, 1 GPU).  Each ncu command runs
# only after the same command exited 0 without ncu.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
B="python bench.py --steps 20 --warmup 5 --clock-window 0.2 --no-cpu-baseline"
$B > $OUT/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $OUT/launches_n1.csv $B > $OUT/ncu_launches.log 2>&1
V1="python tools/prof_virtual.py --n 1 --iters 8"
$V1 > $OUT/v1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:solo -s 5 -c 1 -o $OUT/solo_n1 $V1 > $OUT/ncu_fused_n1.log 2>&1
V2="python tools/prof_virtual.py --n 2 --iters 5"
$V2 > $OUT/v2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o $OUT/fused_v2 $V2 > $OUT/ncu_fused_v2.log 2>&1
echo done

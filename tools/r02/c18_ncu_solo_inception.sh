#!/bin/bash
set -u
O=gpurun_out/ncu18
mkdir -p $O
for dt in bf16 f32; do
  V="python tools/prof_virtual.py --n 1 --model inception_v3 --dtype $dt --iters 6"
  $V > $O/plain_$dt.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:solo -s 4 -c 1 -o $O/solo_incep_$dt $V > $O/ncu_$dt.log 2>&1
done

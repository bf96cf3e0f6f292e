#!/bin/bash
# N = 1: tile-per-CTA solo kernel (default) vs the persistent bulk-copy variant
# (HVD_CFG_SOLO_KERNEL=1) at several stage geometries, on the bench step and Inception V3.
set -u
O=gpurun_out/c44
mkdir -p $O
for cfg in "" "SOLO_KERNEL=1" "SOLO_KERNEL=1 SOLO_STAGES=4 SOLO_STAGE_BYTES=16384" "SOLO_KERNEL=1 SOLO_STAGES=8 SOLO_STAGE_BYTES=16384" "SOLO_KERNEL=1 SOLO_STAGES=3 SOLO_STAGE_BYTES=65536" "SOLO_KERNEL=1 SOLO_STAGES=6 SOLO_STAGE_BYTES=8192" ""; do
  args=""
  for kv in $cfg; do args="$args --config $kv"; done
  tag=$(echo "x$cfg" | tr ' =' '__')
  for w in fp32_64MiB inception_v3_bf16; do
    timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 200 --warmup 20 $args > $O/${w}_${tag}_$(date +%s%N).log 2>&1
  done
done

#!/bin/bash
# Per-slice device timelines of the 64 MiB registered step at N = 4 under different knobs
# (mean wait between a channel's slices = exposed hop latency), and N = 1 bench lines of
# the model sets.
set -u
O=gpurun_out/tl
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for cfg in "" "PACE_GBPS=700" "PACE_GBPS=650" "CHANNELS=64" "WINDOW=0" "WINDOW=4"; do
  i=$((i+1))
  args=""
  for kv in $cfg; do args="$args --config $kv"; done
  timeout 200 $R --nproc-per-node 4 --master-port $((29680+i)) tools/timeline_capture.py --registered --mib 64 $args --out $O/n4_cfg$i.json > $O/n4_cfg$i.log 2>&1
  echo "cfg$i: $cfg" >> $O/index.txt
done
for w in inception_v3 inception_v3_bf16 resnet101 vgg16 fp32_64MiB; do
  CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 100 --warmup 10 > $O/bench_n1_$w.log 2>&1
done

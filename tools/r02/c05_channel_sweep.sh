#!/bin/bash
# Channel-count sweep of the fused push at 64 MiB (fewer pushing SMs -> shorter NVLink
# store queue -> shorter fence/arrival latency?), N = 4 then N = 2.
set -u
O=gpurun_out/sweep
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P=""
for c in 16 24 32 40 48 64 80 96 128; do
  for w in 2 0 4; do P="$P CHANNELS=$c,WINDOW=$w"; done
done
P="$P CHANNELS=32,SLICE_BYTES=131072 CHANNELS=48,SLICE_BYTES=131072 CHANNELS=64,SLICE_BYTES=131072 CHANNELS=32,SLICE_BYTES=32768 CHANNELS=48,SLICE_BYTES=32768 CHANNELS=64,SLICE_BYTES=32768 LL128_MAX_BYTES=67108864"
timeout 900 $R --nproc-per-node 4 --master-port 29631 tools/sweep_bulk.py --mib 64 16 --iters 40 --points $P --out $O/chan_n4.json > $O/chan_n4.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $R --nproc-per-node 2 --master-port 29632 tools/sweep_bulk.py --mib 64 --iters 40 --points $P --out $O/chan_n2.json > $O/chan_n2.log 2>&1

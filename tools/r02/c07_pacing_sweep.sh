#!/bin/bash
# Remote-store pacing sweep of the fused push at 64 MiB, N = 4 then N = 2.
set -u
O=gpurun_out/sweep
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P="PACE_GBPS=0"
for g in 560 600 640 670 700 730 760 800; do
  for b in 2 8; do P="$P PACE_GBPS=$g,PACE_BURST_ROWS=$b"; done
  P="$P PACE_GBPS=$g,WINDOW=0"
done
P="$P PACE_GBPS=0"
timeout 900 $R --nproc-per-node 4 --master-port 29651 tools/sweep_bulk.py --mib 64 --iters 40 --points $P --out $O/pace_n4.json > $O/pace_n4.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $R --nproc-per-node 2 --master-port 29652 tools/sweep_bulk.py --mib 64 --iters 40 --points $P --out $O/pace_n2.json > $O/pace_n2.log 2>&1
timeout 300 $R --nproc-per-node 4 --master-port 29653 tools/e2e_probe.py > $O/e2e_n4.log 2>&1

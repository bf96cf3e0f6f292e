#!/bin/bash
# Remote-store pacing (globaltimer-based) sweep of the fused push at 64 MiB, N = 4 then N = 2.
set -u
O=gpurun_out/sweep
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P="PACE_GBPS=0"
for g in 620 660 690 710 730 760; do
  for b in 2 8 32; do P="$P PACE_GBPS=$g,PACE_BURST_ROWS=$b"; done
done
P="$P PACE_GBPS=0"
timeout 900 $R --nproc-per-node 4 --master-port 29691 tools/sweep_bulk.py --mib 64 --iters 40 --points $P --out $O/pace2_n4.json > $O/pace2_n4.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $R --nproc-per-node 2 --master-port 29692 tools/sweep_bulk.py --mib 64 --iters 40 --points $P --out $O/pace2_n2.json > $O/pace2_n2.log 2>&1

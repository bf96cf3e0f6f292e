#!/bin/bash
# Slice / window sweep of the fused push with PREISSUE on (default for N > 2).
set -u
O=gpurun_out/c33
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P="SLICE_BYTES=0"
for sl in 32768 49152 65536 98304 131072; do
  for w in 2 3 4 0; do P="$P SLICE_BYTES=$sl,WINDOW=$w"; done
done
P="$P SLICE_BYTES=0"
timeout 900 $R --nproc-per-node 4 --master-port 29841 tools/sweep_bulk.py --mib 64 --max-sets 16 --iters 40 --points $P --out $O/sw_n4.json > $O/sw_n4.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $R --nproc-per-node 2 --master-port 29842 tools/sweep_bulk.py --mib 64 --max-sets 16 --iters 40 --points $P PREISSUE=1 PREISSUE=1,SLICE_BYTES=65536,WINDOW=3 --out $O/sw_n2.json > $O/sw_n2.log 2>&1

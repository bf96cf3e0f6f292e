#!/bin/bash
# A/B of the LL128 line layout on one box: 7/8 (ab/old) vs 15/16 (tree), alternating.
set -u
O=gpurun_out/c23
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P="LL128_MAX_BYTES=33554432"
i=0
for rep in 1 2; do
  for v in old new; do
    i=$((i+1))
    root=""; [ $v = old ] && root=$PWD/ab/old
    CUDA_VISIBLE_DEVICES=0,1 HVD_PKG_ROOT=$root timeout 600 $R --nproc-per-node 2 --master-port $((29740+i)) tools/sweep_bulk.py --mib 1 2 4 8 16 --max-sets 16 --iters 50 --points $P --out $O/${v}_n2_$rep.json > $O/${v}_n2_$rep.log 2>&1
    HVD_PKG_ROOT=$root timeout 600 $R --nproc-per-node 4 --master-port $((29760+i)) tools/sweep_bulk.py --mib 1 2 4 8 16 32 --max-sets 16 --iters 50 --points $P --out $O/${v}_n4_$rep.json > $O/${v}_n4_$rep.log 2>&1
  done
done

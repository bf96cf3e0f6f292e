#!/bin/bash
# LL128 (15/16 layout) vs the fused push around the crossover.
set -u
O=gpurun_out/c24
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P="LL128_MAX_BYTES=0 LL128_MAX_BYTES=67108864 LL128_MAX_BYTES=0 LL128_MAX_BYTES=67108864"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R --nproc-per-node 2 --master-port 29781 tools/sweep_bulk.py --mib 8 12 16 24 32 --max-sets 16 --iters 50 --points $P --out $O/x_n2.json > $O/x_n2.log 2>&1
timeout 600 $R --nproc-per-node 4 --master-port 29782 tools/sweep_bulk.py --mib 16 24 32 48 64 --max-sets 16 --iters 50 --points $P --out $O/x_n4.json > $O/x_n4.log 2>&1

#!/bin/bash
# Bulk (TMA) push with two CTAs per SM (up to 256 channels), as the TMA push probe that
# reached 744 GB/s used; N = 2 then N = 4, 64 MiB registered.
set -u
O=gpurun_out/sweep
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P="PROTOCOL=1"
for ch in 148 256; do
  for sb in "2 16384" "2 32768" "4 16384"; do
    set -- $sb
    for d in 1 2; do
      for sl in 65536 131072; do
        P="$P PROTOCOL=2,BULK_CHANNELS=$ch,BULK_STAGES=$1,BULK_STAGE_BYTES=$2,BULK_DEPTH=$d,BULK_SLICE_BYTES=$sl"
      done
    done
  done
done
P="$P PROTOCOL=1"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $R --nproc-per-node 2 --master-port 29701 tools/sweep_bulk.py --mib 64 --iters 40 --points $P --out $O/bulk2_n2.json > $O/bulk2_n2.log 2>&1
timeout 900 $R --nproc-per-node 4 --master-port 29702 tools/sweep_bulk.py --mib 64 --iters 40 --points $P --out $O/bulk2_n4.json > $O/bulk2_n4.log 2>&1

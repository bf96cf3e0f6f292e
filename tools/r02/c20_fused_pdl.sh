#!/bin/bash
# Programmatic dependent launch of the fused push: back-to-back 64 MiB / 8 MiB calls.
set -u
O=gpurun_out/sweep
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P="FUSED_PDL=0 FUSED_PDL=1 FUSED_PDL=2 FUSED_PDL=0 FUSED_PDL=1 FUSED_PDL=2 LL128_MAX_BYTES=0,FUSED_PDL=0 LL128_MAX_BYTES=0,FUSED_PDL=1 LL128_MAX_BYTES=0,FUSED_PDL=2"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R --nproc-per-node 2 --master-port 29711 tools/sweep_bulk.py --mib 64 8 --iters 50 --points $P --out $O/pdl_n2.json > $O/pdl_n2.log 2>&1
timeout 600 $R --nproc-per-node 4 --master-port 29712 tools/sweep_bulk.py --mib 64 8 --iters 50 --points $P --out $O/pdl_n4.json > $O/pdl_n4.log 2>&1

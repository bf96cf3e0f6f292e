#!/bin/bash
# LL / LL128 programmatic dependent launch A/B: small and mid sizes back to back.
set -u
O=gpurun_out/c34
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x -k "pdl or ll or knobs" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
P="LL_PDL=0 LL_PDL=1 LL_PDL=0 LL_PDL=1"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R --nproc-per-node 2 --master-port 29851 tools/sweep_bulk.py --mib 0.001 0.0625 0.25 1 4 16 --max-sets 16 --iters 200 --points $P --out $O/pdl_n2.json > $O/pdl_n2.log 2>&1
timeout 600 $R --nproc-per-node 4 --master-port 29852 tools/sweep_bulk.py --mib 0.001 0.0625 0.25 1 4 16 --max-sets 16 --iters 200 --points $P --out $O/pdl_n4.json > $O/pdl_n4.log 2>&1

#!/bin/bash
# PREISSUE A/B (fused push), same box, alternating; plus bit-exactness tests.
set -u
O=gpurun_out/c32
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x -k "knobs or registered or model or bitexact or fusion_off or many" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
P="PREISSUE=0 PREISSUE=1 PREISSUE=0 PREISSUE=1 PREISSUE=0 PREISSUE=1 LL128_MAX_BYTES=0,PREISSUE=0 LL128_MAX_BYTES=0,PREISSUE=1"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R --nproc-per-node 2 --master-port 29831 tools/sweep_bulk.py --mib 64 32 --max-sets 16 --iters 50 --points $P --out $O/p_n2.json > $O/p_n2.log 2>&1
timeout 600 $R --nproc-per-node 4 --master-port 29832 tools/sweep_bulk.py --mib 64 --max-sets 16 --iters 50 --points $P --out $O/p_n4.json > $O/p_n4.log 2>&1

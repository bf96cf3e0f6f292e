#!/bin/bash
# Dependency watcher A/B (fused push), same box, alternating.
set -u
O=gpurun_out/c30
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_virtual.py -q -x -k "knobs or registered or model or bench" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
P="WATCHER=0 WATCHER=1 WATCHER=0 WATCHER=1 LL128_MAX_BYTES=0,WATCHER=0 LL128_MAX_BYTES=0,WATCHER=1 LL128_MAX_BYTES=0,WATCHER=0 LL128_MAX_BYTES=0,WATCHER=1"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R --nproc-per-node 2 --master-port 29801 tools/sweep_bulk.py --mib 64 16 --max-sets 16 --iters 50 --points $P --out $O/w_n2.json > $O/w_n2.log 2>&1
timeout 600 $R --nproc-per-node 4 --master-port 29802 tools/sweep_bulk.py --mib 64 16 --max-sets 16 --iters 50 --points $P --out $O/w_n4.json > $O/w_n4.log 2>&1

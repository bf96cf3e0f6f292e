#!/bin/bash
set -u
O=gpurun_out/c22
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_virtual.py tests/test_gpu_bulk.py -q -x -k "ll128 or model or bench_step or selftest or mixed or host or fusion_off" > $O/pytest_v.log 2>&1; echo rc=$? >> $O/pytest_v.log
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -q -x > $O/pytest_mp.log 2>&1; echo rc=$? >> $O/pytest_mp.log
P="LL128_MAX_BYTES=33554432"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R --nproc-per-node 2 --master-port 29731 tools/sweep_bulk.py --mib 1 2 4 8 16 --iters 50 --points $P --out $O/ll128_n2.json > $O/ll128_n2.log 2>&1
timeout 600 $R --nproc-per-node 4 --master-port 29732 tools/sweep_bulk.py --mib 1 2 4 8 16 32 --iters 50 --points $P --out $O/ll128_n4.json > $O/ll128_n4.log 2>&1

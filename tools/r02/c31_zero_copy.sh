#!/bin/bash
set -u
O=gpurun_out/c31
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x -k "host or solo" > $O/pytest_v.log 2>&1; echo rc=$? >> $O/pytest_v.log
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -q -x -k "oracle" > $O/pytest_mp.log 2>&1; echo rc=$? >> $O/pytest_mp.log
timeout 300 python tools/e2e_probe.py > /dev/null 2>&1 || true
timeout 300 python bench.py --no-cpu-baseline --steps 100 --warmup 10 > $O/bench_n1.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $R --nproc-per-node 2 --master-port 29811 bench.py --gpus 2 --steps 100 --warmup 10 > $O/bench_n2.log 2>&1
timeout 300 $R --nproc-per-node 4 --master-port 29812 bench.py --gpus 4 --steps 100 --warmup 10 > $O/bench_n4.log 2>&1

#!/bin/bash
set -u
O=gpurun_out/b42
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R --nproc-per-node 2 --master-port 29891 bench.py --gpus 2 > $O/bench_n2.log 2>&1
timeout 600 $R --nproc-per-node 4 --master-port 29892 bench.py --gpus 4 > $O/bench_n4.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R --nproc-per-node 2 --master-port 29893 bench.py --gpus 2 --impl reference --steps 3 --warmup 3 > $O/bench_reference_n2.log 2>&1

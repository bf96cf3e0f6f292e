#!/bin/bash
# After the device-memory error word: e2e probe at N = 2 and 4, GPU tests (4 GPUs).
set -u
O=gpurun_out/c9
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $R --nproc-per-node 2 --master-port 29671 tools/e2e_probe.py > $O/e2e_n2.log 2>&1
timeout 300 $R --nproc-per-node 4 --master-port 29672 tools/e2e_probe.py > $O/e2e_n4.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log

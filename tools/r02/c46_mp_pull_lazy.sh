#!/bin/bash
# Lazy pull buffers at 2 GPUs: the multi-process suite (protocols 1/0/2, pull_buffers on
# for 0) and the N=2 bench line.
mkdir -p gpurun_out/c46
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -m gpu -x -q -p no:cacheprovider > gpurun_out/c46/pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/c46/pytest.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 > gpurun_out/c46/bench_n2.log 2>&1
tail -3 gpurun_out/c46/pytest.log
grep '^{' gpurun_out/c46/bench_n2.log | tail -1 | cut -c1-250

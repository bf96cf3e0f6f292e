#!/bin/bash
# Round-2 re-entry check on a 2-GPU box: GPU tests, N=1 and N=2 bench lines.
set -u
O=gpurun_out/chk
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
timeout 300 python bench.py > $O/bench_n1.log 2>&1
timeout 300 $R --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 > $O/bench_n2.log 2>&1
echo done > $O/DONE

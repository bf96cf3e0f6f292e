#!/bin/bash
set -u
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 1 2 4; do
  timeout 400 $R --nproc-per-node $n --master-port $((29860+n)) tools/e2e_probe.py > gpurun_out/e2e36_n$n.log 2>&1
done

#!/bin/bash
# Launch boundary of the bench step: kernel duration, inter-kernel gap, op span (N = 2, 4).
mkdir -p gpurun_out/c48
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29640 + n)) tools/boundary_probe.py > gpurun_out/c48/n$n.log 2>&1
  grep pdl= gpurun_out/c48/n$n.log | cut -c1-900
  tail -3 gpurun_out/c48/n$n.log | grep -i error
done

#!/bin/bash
# Registered vs plain-tensor 64 MiB allreduce: final-scatter cost, FIN_LAG / slice / channel variants.
mkdir -p gpurun_out/c47
for n in 2 4; do
  [ "$(nvidia-smi -L | wc -l)" -ge $n ] || continue
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29600 + n)) tools/nonreg_probe.py > gpurun_out/c47/n$n.log 2>&1
  grep -v '^{' gpurun_out/c47/n$n.log | tail -20
done

#!/bin/bash
set -u
O=gpurun_out/nvlink
mkdir -p $O
python tools/nvml_probe.py > $O/nvml_probe.log 2>&1
for m in 0 1 2; do
  timeout 120 ncu --metrics gpu__time_duration.sum -c 10 python tools/ncu_min.py $m > $O/ncu_min_$m.log 2>&1; echo rc=$? >> $O/ncu_min_$m.log
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 tools/pcie_probe.py > gpurun_out/pcie_n4.log 2>&1

#!/bin/bash
set -u
O=gpurun_out/c15
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_virtual.py -q -x -k "solo or n1 or model or negotiated" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for w in inception_v3 inception_v3_bf16 resnet101 fp32_64MiB; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 100 --warmup 10 > $O/bench_n1_$w.log 2>&1
done

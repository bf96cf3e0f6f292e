#!/bin/bash
set -u
O=gpurun_out/c19
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_virtual.py tests/test_gpu_bulk.py tests/test_gpu_timeline.py -q -x > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for w in inception_v3 inception_v3_bf16 resnet101 vgg16 fp32_64MiB; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 100 --warmup 10 > $O/bench_n1_$w.log 2>&1
done

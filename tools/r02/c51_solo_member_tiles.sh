#!/bin/bash
# Solo kernel: member tiles built with the plan (one descriptor per tile).  GPU suite, then the
# N = 1 bench lines of every workload (two passes, alternating).
mkdir -p gpurun_out/c51
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c51/pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/c51/pytest.log
tail -3 gpurun_out/c51/pytest.log
for pass in 1 2; do
  for w in fp32_64MiB inception_v3 inception_v3_bf16 resnet101 vgg16; do
    timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/c51/bench_${w}_p$pass.log 2>&1
    python -c "
import json,sys
d=json.loads([l for l in open('gpurun_out/c51/bench_${w}_p$pass.log') if l.startswith('{')][-1])
print('$w', $pass, round(d['value'],1), round(d['roofline']['frac'],3), round(d['ms_per_step']*1e3,2), d['clocks'].get('sm_mhz'))"
  done
done

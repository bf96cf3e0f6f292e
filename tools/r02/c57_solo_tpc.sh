#!/bin/bash
# Solo member tiles per CTA A/B: 1 (tree; descriptors now read before griddepcontrol.wait)
# vs 2 / 3 (ab/t2, ab/t3 built with HVD_NVCC_EXTRA=-DHVD_SOLO_TPC=...), alternating; parity
# tests of the solo paths in each variant first.
mkdir -p gpurun_out/c57
for v in tree t2 t3; do
  d=$PWD; [ $v != tree ] && d=$PWD/ab/$v
  (cd $d && timeout 600 python -m pytest tests/test_gpu_virtual.py -m gpu -x -q -k "solo or model_gradient_sets or allreduce_host" -p no:cacheprovider) > gpurun_out/c57/pytest_$v.log 2>&1
  echo "$v pytest exit $?"; tail -1 gpurun_out/c57/pytest_$v.log
done
for pass in 1 2; do
  for v in tree t2 t3; do
    d=$PWD; [ $v != tree ] && d=$PWD/ab/$v
    for w in fp32_64MiB inception_v3 inception_v3_bf16 resnet101; do
      (cd $d && timeout 300 python bench.py --workload $w --no-cpu-baseline) > gpurun_out/c57/${v}_${w}_p$pass.log 2>&1
      python -c "
import json
d=json.loads([l for l in open('gpurun_out/c57/${v}_${w}_p$pass.log') if l.startswith('{')][-1])
print('$v', '$w', $pass, round(d['value'],1), round(d['roofline']['frac'],3), round(d['ms_per_step']*1e3,2))"
    done
  done
done

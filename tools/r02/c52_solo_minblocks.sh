#!/bin/bash
# Solo kernel register cap A/B: default (52 regs, 9 CTAs/SM) vs __launch_bounds__ min 12 / 16
# CTAs per SM (ab/minb12, ab/minb16 built with HVD_NVCC_EXTRA=-DHVD_SOLO_MINB=...), alternating.
mkdir -p gpurun_out/c52
for pass in 1 2; do
  for v in tree minb12 minb16; do
    d=$PWD; [ $v != tree ] && d=$PWD/ab/$v
    for w in fp32_64MiB inception_v3 inception_v3_bf16; do
      (cd $d && timeout 300 python bench.py --workload $w --no-cpu-baseline) > gpurun_out/c52/${v}_${w}_p$pass.log 2>&1
      python -c "
import json
d=json.loads([l for l in open('gpurun_out/c52/${v}_${w}_p$pass.log') if l.startswith('{')][-1])
print('$v', '$w', $pass, round(d['value'],1), round(d['roofline']['frac'],3), round(d['ms_per_step']*1e3,2))"
    done
  done
done

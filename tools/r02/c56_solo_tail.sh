#!/bin/bash
# Solo member tiles: HVD_CFG_SOLO_TAIL A/B (0 = off, -1 = one wave halved, 2664 = two waves,
# 1048576 = every tile halved), same box, alternating; then the new parity tests.
mkdir -p gpurun_out/c56
timeout 600 python -m pytest tests/test_gpu_virtual.py -m gpu -x -q -k "solo" -p no:cacheprovider > gpurun_out/c56/pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/c56/pytest.log
tail -2 gpurun_out/c56/pytest.log
for pass in 1 2; do
  for t in 0 -1 2664 1048576; do
    for w in fp32_64MiB inception_v3 inception_v3_bf16; do
      timeout 300 python bench.py --workload $w --no-cpu-baseline --config SOLO_TAIL=$t > gpurun_out/c56/t${t}_${w}_p$pass.log 2>&1
      python -c "
import json
d=json.loads([l for l in open('gpurun_out/c56/t${t}_${w}_p$pass.log') if l.startswith('{')][-1])
print('$t', '$w', $pass, round(d['value'],1), round(d['roofline']['frac'],3), round(d['ms_per_step']*1e3,2))"
    done
  done
done

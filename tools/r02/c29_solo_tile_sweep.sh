#!/bin/bash
# N = 1 solo kernel tile geometry sweep (builds variants in the box's copy of the tree).
set -u
O=gpurun_out/solo29
mkdir -p $O
for cfg in ${SOLO_CFGS:-128x8}; do
  set -- ${cfg/x/ }
  tag=t$1_u$2
  HVD_NVCC_EXTRA="-DHVD_SOLO_THREADS=$1 -DHVD_SOLO_U=$2" python -c "
import importlib.util
spec=importlib.util.spec_from_file_location('b','paper_1802_05799_b200/_build.py'); m=importlib.util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > $O/build_$tag.log 2>&1 || continue
  for w in ${SOLO_WORKLOADS:-fp32_64MiB inception_v3_bf16}; do
    timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 200 --warmup 20 > $O/bench_${tag}_${w}_$(date +%s%N).log 2>&1
  done
done

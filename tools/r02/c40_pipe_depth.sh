#!/bin/bash
# cp.async prefetch depth (kPipe rows per data thread) of the fused push: builds variants in
# the box's copy of the tree, bench lines at N = 2 and 4.
set -u
O=gpurun_out/pipe40
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for p in 8 4 6 12 8; do
  HVD_NVCC_EXTRA="-DHVD_PIPE=$p" python -c "
import importlib.util
spec=importlib.util.spec_from_file_location('b','paper_1802_05799_b200/_build.py'); m=importlib.util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > $O/build_$p.log 2>&1 || continue
  ts=$(date +%s%N)
  CUDA_VISIBLE_DEVICES=0,1 timeout 300 $R --nproc-per-node 2 --master-port 29881 bench.py --gpus 2 --steps 100 --warmup 10 --no-cpu-baseline > $O/n2_p${p}_$ts.log 2>&1
  timeout 300 $R --nproc-per-node 4 --master-port 29882 bench.py --gpus 4 --steps 100 --warmup 10 --no-cpu-baseline > $O/n4_p${p}_$ts.log 2>&1
done

#!/bin/bash
# Fused push: odd channels staggered (HVD_CFG_STAGGER_NS) at N = 4 and 2, bench step
# (registered fp32) at 64 / 128 MiB, two alternating passes.
mkdir -p gpurun_out/c59
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P="STAGGER_NS=0 STAGGER_NS=3000 STAGGER_NS=6000 STAGGER_NS=12000 STAGGER_NS=0"
i=0
for rep in 1 2; do
  i=$((i+1))
  timeout 600 $R --nproc-per-node 4 --master-port $((29600+i)) tools/sweep_bulk.py --mib 64 128 --iters 60 --points $P --out gpurun_out/c59/n4_$rep.json > gpurun_out/c59/n4_$rep.log 2>&1
  CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R --nproc-per-node 2 --master-port $((29610+i)) tools/sweep_bulk.py --mib 64 128 --iters 60 --points $P --out gpurun_out/c59/n2_$rep.json > gpurun_out/c59/n2_$rep.log 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/c59/n*_*.json')):
    for r in json.load(open(f)):
        print(f.split('/')[-1], r['point'], r['mib'], round(r['busbw'], 1), round(r['us'], 1), r.get('bitexact_vs_first_point'))
PY

#!/bin/bash
# Fine channel-count sweep around the default 128 (bench step, 64 / 256 MiB), N = 4 and 2.
mkdir -p gpurun_out/c63
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P="CHANNELS=128 CHANNELS=112 CHANNELS=120 CHANNELS=136 CHANNELS=144 CHANNELS=128"
i=0
for rep in 1 2; do
  i=$((i+1))
  timeout 600 $R --nproc-per-node 4 --master-port $((29660+i)) tools/sweep_bulk.py --mib 64 256 --iters 60 --points $P --out gpurun_out/c63/n4_$rep.json > gpurun_out/c63/n4_$rep.log 2>&1
  CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R --nproc-per-node 2 --master-port $((29670+i)) tools/sweep_bulk.py --mib 64 256 --iters 60 --points $P --out gpurun_out/c63/n2_$rep.json > gpurun_out/c63/n2_$rep.log 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/c63/n*_*.json')):
    for r in json.load(open(f)):
        print(f.split('/')[-1], r['point'], r['mib'], round(r['busbw'], 1), round(r['us'], 1), r.get('bitexact_vs_first_point'))
PY

#!/bin/bash
# Bench step at sizes just below 64 MiB (N = 2): is the drop from 64 to 62.9 MiB smooth in
# size, or does only the power of two run at full rate (alignment of the channel shares)?
mkdir -p gpurun_out/c67
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R --nproc-per-node 2 --master-port 29851 tools/sweep_bulk.py --mib 62.9 63 63.5 63.75 63.9921875 64 64.0078125 65 --iters 60 --points CHANNELS=128 --out gpurun_out/c67/n2.json > gpurun_out/c67/n2.log 2>&1
python - <<'PY'
import json
for r in json.load(open('gpurun_out/c67/n2.json')):
    print(r['mib'], round(r['busbw'], 1), round(r['us'], 1))
PY

#!/bin/bash
# A call just over the 64 MiB fusion capacity (a 64 MiB buffer + a small tail buffer): the tail
# in its own LL launch (default) vs inside the fused multi-buffer launch (LL_MAX_BYTES=0),
# N = 2 and 4.
mkdir -p gpurun_out/c68
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P="LL_MAX_BYTES=262144 LL_MAX_BYTES=0 LL_MAX_BYTES=262144"
timeout 600 $R --nproc-per-node 4 --master-port 29861 tools/sweep_bulk.py --mib 64 64.0078125 64.25 65 --iters 60 --points $P --out gpurun_out/c68/n4.json > gpurun_out/c68/n4.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R --nproc-per-node 2 --master-port 29862 tools/sweep_bulk.py --mib 64 64.0078125 64.25 65 --iters 60 --points $P --out gpurun_out/c68/n2.json > gpurun_out/c68/n2.log 2>&1
python - <<'PY'
import json
for n in (2, 4):
    for r in json.load(open(f'gpurun_out/c68/n{n}.json')):
        print(n, r['point'], r['mib'], round(r['busbw'], 1), round(r['us'], 1), r['kernels'], r.get('bitexact_vs_first_point'))
PY

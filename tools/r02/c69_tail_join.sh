#!/bin/bash
# Small buffers join the fused launch of a few-buffer plan: the GPU suite (4 GPUs), the tail
# buffer sizes at N = 2 / 4, and the model sets C2-C4 at N = 4.
mkdir -p gpurun_out/c69
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c69/pytest.log 2>&1
echo "pytest exit $?"; tail -1 gpurun_out/c69/pytest.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $R --nproc-per-node 4 --master-port 29871 tools/sweep_bulk.py --mib 64 64.0078125 64.25 65 --iters 60 --points LL_MAX_BYTES=262144 --out gpurun_out/c69/n4.json > gpurun_out/c69/n4.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R --nproc-per-node 2 --master-port 29872 tools/sweep_bulk.py --mib 64 64.0078125 64.25 65 --iters 60 --points LL_MAX_BYTES=262144 --out gpurun_out/c69/n2.json > gpurun_out/c69/n2.log 2>&1
timeout 900 $R --nproc-per-node 4 --master-port 29873 tools/bench_configs.py --only C2,C3,C4 --no-nccl --iters 20 --out gpurun_out/c69/cfg_n4.json > gpurun_out/c69/cfg_n4.log 2>&1
python - <<'PY'
import json
for n in (2, 4):
    for r in json.load(open(f'gpurun_out/c69/n{n}.json')):
        print(n, r['point'], r['mib'], round(r['busbw'], 1), round(r['us'], 1), r['kernels'], r.get('bitexact_vs_first_point'))
d=json.load(open('gpurun_out/c69/cfg_n4.json'))
print(' '.join(f"{r['config']}{r.get('model','')[:4]}{r['dtype']}t{int(r['fusion_threshold']>0)}={r['us_per_allreduce']:.1f}/{r.get('launches_per_call')}" for r in d['rows'] if r['config'] in ('C2','C3','C4')))
PY

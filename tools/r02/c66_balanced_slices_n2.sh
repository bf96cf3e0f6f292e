#!/bin/bash
# Equal slices at N = 2: tree vs ab/prev (8ed227f, before the change), same box, alternating:
# model sets C2-C4 and the bench step at 62.9 / 48.3 MiB.
mkdir -p gpurun_out/c66
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
TOP=$PWD
i=0
for rep in 1 2; do
  for v in tree prev; do
    i=$((i+1))
    root=""; d=$PWD; [ $v = prev ] && root=$PWD/ab/prev && d=$PWD/ab/prev
    HVD_PKG_ROOT=$root timeout 600 $R --nproc-per-node 2 --master-port $((29800+i)) tools/sweep_bulk.py --mib 62.9 48.3 --iters 60 --points CHANNELS=128 --out gpurun_out/c66/sw_${v}_n2_$rep.json > gpurun_out/c66/sw_${v}_n2_$rep.log 2>&1
    (cd $d && timeout 900 $R --nproc-per-node 2 --master-port $((29820+i)) tools/bench_configs.py --only C2,C3,C4 --no-nccl --iters 20 --out $TOP/gpurun_out/c66/cfg_${v}_n2_$rep.json) > gpurun_out/c66/cfg_${v}_n2_$rep.log 2>&1
  done
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/c66/sw_*.json')):
    for r in json.load(open(f)):
        print(f.split('/')[-1], r['point'], r['mib'], round(r['busbw'], 1), round(r['us'], 1), r.get('bitexact_vs_first_point'))
for f in sorted(glob.glob('gpurun_out/c66/cfg_*.json')):
    d=json.load(open(f))
    print(f.split('/')[-1], ' '.join(f"{r['config']}{r.get('model','')[:4]}{r['dtype']}t{int(r['fusion_threshold']>0)}={r['us_per_allreduce']:.1f}" for r in d['rows'] if r['config'] in ('C2','C3','C4')))
PY

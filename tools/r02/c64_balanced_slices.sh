#!/bin/bash
# Balanced slices (no runt last slice): GPU suite on the tree, then tree vs ab/prev (HEAD
# before the change) on the same box: channel counts around 128 at 64 MiB and the model
# sets C2-C4 plus C5 from 1 MiB up, N = 4 and 2, alternating.
mkdir -p gpurun_out/c64
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c64/pytest.log 2>&1
echo "pytest exit $?"; tail -1 gpurun_out/c64/pytest.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P="CHANNELS=128 CHANNELS=120 CHANNELS=136 CHANNELS=100"
TOP=$PWD
i=0
for rep in 1 2; do
  for v in tree prev; do
    i=$((i+1))
    root=""; d=$PWD; [ $v = prev ] && root=$PWD/ab/prev && d=$PWD/ab/prev
    HVD_PKG_ROOT=$root timeout 600 $R --nproc-per-node 4 --master-port $((29700+i)) tools/sweep_bulk.py --mib 64 48.3 --iters 60 --points $P --out gpurun_out/c64/sw_${v}_n4_$rep.json > gpurun_out/c64/sw_${v}_n4_$rep.log 2>&1
    (cd $d && timeout 900 $R --nproc-per-node 4 --master-port $((29720+i)) tools/bench_configs.py --only C2,C3,C4,C5 --sweep-min-log2 20 --no-nccl --iters 20 --out $TOP/gpurun_out/c64/cfg_${v}_n4_$rep.json) > gpurun_out/c64/cfg_${v}_n4_$rep.log 2>&1
    (cd $d && CUDA_VISIBLE_DEVICES=0,1 timeout 900 $R --nproc-per-node 2 --master-port $((29740+i)) tools/bench_configs.py --only C2,C3,C4,C5 --sweep-min-log2 20 --no-nccl --iters 20 --out $TOP/gpurun_out/c64/cfg_${v}_n2_$rep.json) > gpurun_out/c64/cfg_${v}_n2_$rep.log 2>&1
  done
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/c64/sw_*.json')):
    for r in json.load(open(f)):
        print(f.split('/')[-1], r['point'], r['mib'], round(r['busbw'], 1), round(r['us'], 1), r.get('bitexact_vs_first_point'))
for f in sorted(glob.glob('gpurun_out/c64/cfg_*.json')):
    d=json.load(open(f))
    out=[]
    for r in d['rows']:
        if r['config'] in ('C2','C3','C4'): out.append(f"{r['config']}{r.get('model','')[:4]}{r['dtype']}t{r['fusion_threshold']>0:d}={r['us_per_allreduce']:.1f}")
        elif r['config']=='C5' and r['dtype']=='f32' and r['bytes'] in (1<<20, 64<<20, 1<<30): out.append(f"C5 {r['bytes']>>20}M={r['us']:.1f}")
    print(f.split('/')[-1], ' '.join(out))
PY

#!/bin/bash
# Fused push kernel capped at 112 registers (ab/r112, HVD_FUSED_MAXNREG=112: two CTAs fit on
# an SM, so the next launch can become resident under programmatic dependent launch) vs
# the tree (124-128 registers), FUSED_PDL 0 / 1 / 2, bench step at 64 MiB, N = 2 and 4.
mkdir -p gpurun_out/c61
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P="FUSED_PDL=0 FUSED_PDL=1 FUSED_PDL=2 FUSED_PDL=0"
i=0
for rep in 1 2; do
  for v in tree r112; do
    i=$((i+1))
    root=""; [ $v = r112 ] && root=$PWD/ab/r112
    HVD_PKG_ROOT=$root timeout 600 $R --nproc-per-node 4 --master-port $((29500+i)) tools/sweep_bulk.py --mib 64 --iters 80 --points $P --out gpurun_out/c61/${v}_n4_$rep.json > gpurun_out/c61/${v}_n4_$rep.log 2>&1
    CUDA_VISIBLE_DEVICES=0,1 HVD_PKG_ROOT=$root timeout 600 $R --nproc-per-node 2 --master-port $((29520+i)) tools/sweep_bulk.py --mib 64 --iters 80 --points $P --out gpurun_out/c61/${v}_n2_$rep.json > gpurun_out/c61/${v}_n2_$rep.log 2>&1
  done
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/c61/*.json')):
    for r in json.load(open(f)):
        print(f.split('/')[-1], r['point'], round(r['busbw'], 1), round(r['us'], 1), r.get('bitexact_vs_first_point'))
PY

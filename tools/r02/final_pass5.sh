#!/bin/bash
# Last pass of the round (gpurun --gpus 4): the whole GPU suite, smoke, bench N = 1 (with the
# CPU baseline) / 2 / 4, the N = 1 reference arm, model sets at N = 1, ncu launch list of
# the N = 1 bench and a full capture of the solo kernel.
set -u
O=gpurun_out/final5
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1700 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > $O/bench_n1.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R --nproc-per-node 2 --master-port 29971 bench.py --gpus 2 > $O/bench_n2.log 2>&1
timeout 600 $R --nproc-per-node 4 --master-port 29972 bench.py --gpus 4 > $O/bench_n4.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference_n1.log 2>&1
for w in resnet101 inception_v3 inception_v3_bf16 vgg16; do
  CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 100 --warmup 10 > $O/bench_n1_$w.log 2>&1
done
B="python bench.py --steps 20 --warmup 5 --clock-window 0.2 --no-cpu-baseline"
CUDA_VISIBLE_DEVICES=0 $B > $O/bench_plain.log 2>&1 && CUDA_VISIBLE_DEVICES=0 timeout 600 \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_n1.csv $B > $O/ncu_launches.log 2>&1
V1="python tools/prof_virtual.py --n 1 --iters 8"
CUDA_VISIBLE_DEVICES=0 $V1 > $O/v1_plain.log 2>&1 && CUDA_VISIBLE_DEVICES=0 timeout 600 \
  ncu --set full --clock-control none --import-source on -k regex:solo -s 5 -c 1 -o $O/solo_n1 $V1 > $O/ncu_solo_n1.log 2>&1
echo done > $O/DONE

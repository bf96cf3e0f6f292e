#!/bin/bash
# End-of-round measurement pass on a 4-GPU box (gpurun --gpus 4): tests, bench lines
# (N = 1, 2, 4 and the reference arm), configs C2-C5, timelines, ncu.  Outputs under
# gpurun_out/final/; copy what is judged into profiles/.
set -u
O=gpurun_out/final
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_n1.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference_n1.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 > $O/bench_n2.log 2>&1
timeout 600 $R --nproc-per-node 4 --master-port 29602 bench.py --gpus 4 > $O/bench_n4.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $R --nproc-per-node 2 --master-port 29603 bench.py --gpus 2 --impl reference --steps 3 --warmup 3 > $O/bench_reference_n2.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $R --nproc-per-node 2 --master-port 29604 tools/bench_configs.py --out $O/configs_n2.json > $O/configs_n2.log 2>&1
timeout 900 $R --nproc-per-node 4 --master-port 29605 tools/bench_configs.py --out $O/configs_n4.json > $O/configs_n4.log 2>&1
for n in 2 4; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((n-1))) timeout 300 $R --nproc-per-node $n --master-port 2961$n tools/timeline_capture.py --registered --out $O/timeline_registered_n$n.json > $O/timeline_n$n.log 2>&1
done
# ncu: launch list of the N = 1 bench, full captures of the N = 1 solo kernel and of the
# fused kernel with 2 ranks simulated on one GPU (a multi-GPU launch cannot be replayed)
B="python bench.py --steps 20 --warmup 5 --clock-window 0.2 --no-cpu-baseline"
CUDA_VISIBLE_DEVICES=0 $B > $O/bench_plain.log 2>&1 && CUDA_VISIBLE_DEVICES=0 timeout 600 \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_n1.csv $B > $O/ncu_launches.log 2>&1
V1="python tools/prof_virtual.py --n 1 --iters 8"
CUDA_VISIBLE_DEVICES=0 $V1 > $O/v1_plain.log 2>&1 && CUDA_VISIBLE_DEVICES=0 timeout 600 \
  ncu --set full --clock-control none --import-source on -k regex:solo -s 5 -c 1 -o $O/solo_n1 $V1 > $O/ncu_solo_n1.log 2>&1
V2="python tools/prof_virtual.py --n 2 --iters 5"
CUDA_VISIBLE_DEVICES=0 $V2 > $O/v2_plain.log 2>&1 && CUDA_VISIBLE_DEVICES=0 timeout 900 \
  ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o $O/fused_v2 $V2 > $O/ncu_fused_v2.log 2>&1
echo done > $O/DONE

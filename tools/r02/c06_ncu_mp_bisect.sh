#!/bin/bash
set -u
O=gpurun_out/ncump
mkdir -p $O
export WORLD_SIZE=2 MASTER_ADDR=127.0.0.1
for m in 3 4 5; do
  export MASTER_PORT=$((29800 + m))
  EXTRA=""
  [ $m = 4 ] && export HVD_NVLINK_CHECK=0
  [ $m = 5 ] && unset HVD_NVLINK_CHECK
  RANK=1 LOCAL_RANK=1 timeout 100 python tools/ncu_mp_min.py $((m>4?4:m)) > $O/r1_$m.log 2>&1 &
  p=$!
  RANK=0 LOCAL_RANK=0 timeout 90 ncu --metrics gpu__time_duration.sum -c 8 python tools/ncu_mp_min.py $((m>4?4:m)) > $O/r0_$m.log 2>&1
  echo rc=$? >> $O/r0_$m.log
  wait $p; echo rc=$? >> $O/r1_$m.log
done
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $R --nproc-per-node 2 --master-port 29641 tools/e2e_probe.py > $O/e2e_n2.log 2>&1

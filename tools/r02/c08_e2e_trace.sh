#!/bin/bash
set -u
O=gpurun_out/ncump
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
E2E_CHUNK_MIB=4 timeout 300 $R --nproc-per-node 2 --master-port 29661 tools/e2e_trace.py > $O/e2e_trace_n2.log 2>&1
E2E_CHUNK_MIB=8 timeout 300 $R --nproc-per-node 2 --master-port 29662 tools/e2e_trace.py > $O/e2e_trace_n2_8.log 2>&1
export WORLD_SIZE=2 MASTER_ADDR=127.0.0.1
for m in 3 5; do
  export MASTER_PORT=$((29810 + m))
  RANK=1 LOCAL_RANK=1 timeout 100 python tools/ncu_mp_min.py $((m>4?4:m)) > $O/d_r1_$m.log 2>&1 &
  p=$!
  RANK=0 LOCAL_RANK=0 timeout 90 ncu --devices 0 --metrics gpu__time_duration.sum -c 8 python tools/ncu_mp_min.py $((m>4?4:m)) > $O/d_r0_$m.log 2>&1
  echo rc=$? >> $O/d_r0_$m.log
  wait $p; echo rc=$? >> $O/d_r1_$m.log
done

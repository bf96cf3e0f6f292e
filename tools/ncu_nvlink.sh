#!/bin/bash
# NVLink counters of the ring kernel on a real N-GPU job: rank 0 under ncu,
# ranks 1..N-1 plain.  Usage: tools/ncu_nvlink.sh N [protocol] [kernel regex] [metrics] [tag]
set -u
N=${1:-2}; P=${2:-1}; K=${3:-fused}; MM=${4:-}; TAG=${5:-}
O=gpurun_out/nvlink
mkdir -p $O
PORT=$((29700 + N + 10 * P))
M=gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvltx__bytes_data_protocol.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvlrx__bytes_data_protocol.sum,dram__bytes_read.sum,dram__bytes_write.sum
[ -n "$MM" ] && M=$MM
export WORLD_SIZE=$N MASTER_ADDR=127.0.0.1 MASTER_PORT=$PORT NVL_PROTOCOL=$P
pids=()
for r in $(seq 1 $((N-1))); do
  RANK=$r LOCAL_RANK=$r timeout 250 python tools/ncu_nvlink.py > $O/rank${r}_n${N}_p${P}${TAG}.log 2>&1 &
  pids+=($!)
done
RANK=0 LOCAL_RANK=0 timeout 240 ncu --metrics $M --clock-control none --cache-control none \
  -k regex:$K -c 12 --csv --log-file $O/ncu_n${N}_p${P}${TAG}.csv python tools/ncu_nvlink.py > $O/rank0_n${N}_p${P}${TAG}.log 2>&1
echo "rank0 rc=$?" >> $O/rank0_n${N}_p${P}${TAG}.log
for p in "${pids[@]}"; do wait $p; done

#!/bin/bash
# NVLink counters (ncu range replay over 10 launches, device 0) of the bench step:
# one registered 64 MiB fp32 gradient, allreduce-average, one process driving N GPUs.
set -u
N=${1:-4}
O=gpurun_out/nvlink
mkdir -p $O
M=gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvltx__bytes_data_protocol.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvlrx__bytes_data_protocol.sum,dram__bytes_read.sum,dram__bytes_write.sum
for cfg in "1 64" "2 64" "1 16"; do
  set -- $cfg
  P=$1; MIB=$2
  NVL_PROTOCOL=$P NVL_MIB=$MIB NVL_TAG=_p${P}_${MIB}MiB timeout 300 python tools/nvlink_1proc.py $N 20 > $O/plain_n${N}_p${P}_${MIB}.log 2>&1 || continue
  NVL_PROTOCOL=$P NVL_MIB=$MIB NVL_TAG=_p${P}_${MIB}MiB_ncu NVL_RANGE=1 NVL_RANGE_DEVS=0 timeout 300 ncu --replay-mode app-range --metrics $M --clock-control none --cache-control none --csv --log-file $O/range_n${N}_p${P}_${MIB}.csv python tools/nvlink_1proc.py $N 10 > $O/range_n${N}_p${P}_${MIB}.log 2>&1
done

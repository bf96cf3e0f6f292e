#!/bin/bash
set -u
O=gpurun_out/nvlink
mkdir -p $O
M=gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvltx__bytes_data_protocol.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvlrx__bytes_data_protocol.sum,dram__bytes_read.sum,dram__bytes_write.sum
i=0
for mode in app-range range; do
  for devs in 0 0,1; do
    for dflag in "--devices 0" ""; do
      i=$((i+1))
      NVL_TAG=_v$i NVL_RANGE=1 NVL_RANGE_DEVS=$devs timeout 150 ncu --replay-mode $mode $dflag --metrics $M --clock-control none --cache-control none --csv --log-file $O/v$i.csv python tools/nvlink_1proc.py 2 10 > $O/v$i.log 2>&1
      echo "mode=$mode devs=$devs dflag=$dflag rc=$?" >> $O/v$i.log
    done
  done
done

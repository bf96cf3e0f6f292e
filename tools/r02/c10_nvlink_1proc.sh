#!/bin/bash
# NVLink counters of the fused ring kernel: one process drives all GPUs (ncu cannot
# profile here while another process uses the GPUs), rank 0's launches profiled.
set -u
N=${1:-2}
O=gpurun_out/nvlink
mkdir -p $O
M=gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvltx__bytes_data_protocol.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvlrx__bytes_data_protocol.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 300 python tools/nvlink_1proc.py $N 20 > $O/oneproc_n$N.log 2>&1; rc=$?; echo rc=$rc >> $O/oneproc_n$N.log
if [ $rc = 0 ]; then
  # application-range replay: the timed loop is one range whose kernels run as usual
  # (kernel replay serialises the ranks' launches: a ring kernel would wait for its peer forever)
  NVL_TAG=_ncu NVL_RANGE=1 timeout 400 ncu --replay-mode app-range --devices 0 --metrics $M --clock-control none --cache-control none --csv --log-file $O/ncu_oneproc_n$N.csv python tools/nvlink_1proc.py $N 10 > $O/ncu_oneproc_n$N.log 2>&1
  echo rc=$? >> $O/ncu_oneproc_n$N.log
fi

#!/bin/bash
# ncu --set full of the fused push on a REAL 4-GPU ring: one process drives all four GPUs,
# application-range replay (the app reruns once per pass; the range = 10 launches).
set -u
O=gpurun_out/full62
mkdir -p $O
NVL_PROTOCOL=1 NVL_MIB=64 NVL_TAG=_full timeout 300 python tools/nvlink_1proc.py 4 10 > $O/plain.log 2>&1 || exit 0
NVL_PROTOCOL=1 NVL_MIB=64 NVL_TAG=_full_ncu NVL_RANGE=1 NVL_RANGE_DEVS=0 timeout 1500 ncu --replay-mode app-range --set full --clock-control none -o $O/fused_range_n4 python tools/nvlink_1proc.py 4 10 > $O/ncu.log 2>&1
echo rc=$? >> $O/ncu.log

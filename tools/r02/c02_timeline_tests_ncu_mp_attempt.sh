#!/bin/bash
set -u
O=gpurun_out/c2
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_timeline.py tests/test_gpu_multiprocess.py -k "timeline or trace" -q -x > $O/pytest_trace.log 2>&1; echo rc=$? >> $O/pytest_trace.log
bash tools/ncu_nvlink.sh 2 1 fused
bash tools/ncu_nvlink.sh 2 2 bulk
echo done > $O/DONE

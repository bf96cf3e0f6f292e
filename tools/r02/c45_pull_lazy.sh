#!/bin/bash
# Lazy pull buffers: the whole 1-GPU suite, then the N=1 bench line.
mkdir -p gpurun_out/c45
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c45/pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/c45/pytest.log
timeout 300 python bench.py > gpurun_out/c45/bench_n1.log 2>&1
tail -3 gpurun_out/c45/pytest.log
tail -1 gpurun_out/c45/bench_n1.log | cut -c1-300

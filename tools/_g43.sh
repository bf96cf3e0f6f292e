timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_n1.log 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 --sets 1 > gpurun_out/bench_n1_sets1.log 2>&1
true

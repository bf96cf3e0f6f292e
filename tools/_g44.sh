timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
for pf in 0 1 2 4 8; do timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --clock-window 0.5 --config SOLO_PREFETCH=$pf > gpurun_out/bench_n1_pf$pf.log 2>&1; done
true

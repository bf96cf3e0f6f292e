timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
CUDA_VISIBLE_DEVICES=0,1 timeout 600 python -m pytest tests/test_gpu_multiprocess.py -m gpu -x -q > gpurun_out/pytest_mp2.log 2>&1; echo rc=$? >> gpurun_out/pytest_mp2.log
CUDA_VISIBLE_DEVICES=0,1,2 timeout 600 python -m pytest tests/test_gpu_multiprocess.py -m gpu -x -q > gpurun_out/pytest_mp3.log 2>&1; echo rc=$? >> gpurun_out/pytest_mp3.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $R --nproc-per-node 2 --master-port 29531 bench.py --gpus 2 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_n2.log 2>&1
timeout 300 $R --nproc-per-node 4 --master-port 29532 bench.py --gpus 4 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_n4.log 2>&1
true

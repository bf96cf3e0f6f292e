set -x
timeout 300 python -m pytest tests/test_gpu_virtual.py -m gpu -x -q -k "ll_protocol or back_to_back or raw_buffer" > gpurun_out/pytest_ll.log 2>&1; echo rc=$? >> gpurun_out/pytest_ll.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 tools/bench_configs.py --only C5 --sweep-max-log2 24 --ll-max 8388608 --out gpurun_out/c5ll_n4.json > gpurun_out/c5ll_n4.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 tools/bench_configs.py --only C5 --sweep-max-log2 24 --ll-max 8388608 --out gpurun_out/c5ll_n2.json > gpurun_out/c5ll_n2.log 2>&1
for s in 1 0; do CUDA_VISIBLE_DEVICES=0,1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 50 --warmup 5 --sets $s > gpurun_out/bench_n2_sets$s.log 2>&1; done
true

#!/bin/bash
# hvd_allreduce_host default chunking: ramped (2 / 6 / 8 ... 8 / ~2 MiB, tree) vs uniform
# 8 MiB (ab/prev), bench e2e at N = 1 and 2, alternating; host-path parity tests first.
mkdir -p gpurun_out/c58
timeout 900 python -m pytest tests/test_gpu_virtual.py -m gpu -x -q -k "allreduce_host" -p no:cacheprovider > gpurun_out/c58/pytest.log 2>&1
echo "pytest exit $?"; tail -1 gpurun_out/c58/pytest.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for pass in 1 2; do
  for v in tree prev; do
    i=$((i+1))
    d=$PWD; [ $v = prev ] && d=$PWD/ab/prev
    (cd $d && CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --no-cpu-baseline) > gpurun_out/c58/${v}_n1_p$pass.log 2>&1
    (cd $d && timeout 300 $R --nproc-per-node 2 --master-port $((29950+i)) bench.py --gpus 2 --no-cpu-baseline) > gpurun_out/c58/${v}_n2_p$pass.log 2>&1
    for n in 1 2; do python -c "
import json
d=json.loads([l for l in open('gpurun_out/c58/${v}_n${n}_p$pass.log') if l.startswith('{')][-1])
print('$v', 'n$n', $pass, round(d['value'],1), 'e2e', round(d['e2e']['value'],2), round(d['e2e']['ms_per_step'],3))"; done
  done
done

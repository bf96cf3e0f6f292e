#!/bin/bash
# N = 2 bench step: this tree vs the tree before the member-tile commits (ab/prev = ea3e60b, before the lazy pull buffers),
# same box, alternating three times.
mkdir -p gpurun_out/c54
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for pass in 1 2 3; do
  for v in tree prev; do
    i=$((i+1))
    d=$PWD; [ $v = prev ] && d=$PWD/ab/prev
    (cd $d && timeout 300 $R --nproc-per-node 2 --master-port $((29900+i)) bench.py --gpus 2 --no-cpu-baseline) > gpurun_out/c54/${v}_p$pass.log 2>&1
    python -c "
import json
d=json.loads([l for l in open('gpurun_out/c54/${v}_p$pass.log') if l.startswith('{')][-1])
print('$v', $pass, round(d['value'],1), round(d['ms_per_step']*1e3,2))"
  done
done

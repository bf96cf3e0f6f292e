#!/bin/bash
set -u
O=gpurun_out/c26
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1700 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 1200 $R --nproc-per-node 4 --master-port 29791 tools/bench_configs.py --out $O/configs_n4.json > $O/configs_n4.log 2>&1
timeout 1200 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log

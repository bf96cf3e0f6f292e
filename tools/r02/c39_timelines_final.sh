#!/bin/bash
# Per-slice device timelines of the registered fused push with the round-2 defaults (PREISSUE
# on for N > 2): 64 MiB and 8 MiB (LL128 off so the fused kernel runs), N = 4 and N = 2.
set -u
O=gpurun_out/tl39
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 $R --nproc-per-node 4 --master-port 29871 tools/timeline_capture.py --registered --mib 64 --out $O/n4_64.json > $O/n4_64.log 2>&1
timeout 300 $R --nproc-per-node 4 --master-port 29872 tools/timeline_capture.py --registered --mib 8 --config LL128_MAX_BYTES=0 --out $O/n4_8.json > $O/n4_8.log 2>&1
timeout 300 $R --nproc-per-node 4 --master-port 29873 tools/timeline_capture.py --registered --mib 64 --config PREISSUE=0 --out $O/n4_64_nopre.json > $O/n4_64_nopre.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $R --nproc-per-node 2 --master-port 29874 tools/timeline_capture.py --registered --mib 64 --out $O/n2_64.json > $O/n2_64.log 2>&1

R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port"
timeout 200 $R 29521 tools/diag_mp.py > gpurun_out/diag_all.log 2>&1
timeout 200 $R 29522 tools/diag_mp.py --cases 8 > gpurun_out/diag_8.log 2>&1
timeout 200 $R 29523 tools/diag_mp.py --cases 4,8 > gpurun_out/diag_48.log 2>&1
timeout 200 $R 29524 tools/diag_mp.py --cases 7,8 > gpurun_out/diag_78.log 2>&1
timeout 200 $R 29525 tools/diag_mp.py --ll-max 0 > gpurun_out/diag_all_noll.log 2>&1
true

# NEXT-1 sweep over row phases: tests + timing vs the one-shot sweep (C, D, a W = 8 shard of D)
bash tools/r02_gpu.sh ${1:-sw} tests/test_gpu_sweep_rows.py tests/test_gpu_nccl_plumbing.py
timeout 900 python tools/sweep_rows_time.py C - 4 16 > gpurun_out/${1:-sw}_C.log 2>&1; cat gpurun_out/${1:-sw}_C.log
timeout 1200 python tools/sweep_rows_time.py D - 8 32 > gpurun_out/${1:-sw}_D.log 2>&1; cat gpurun_out/${1:-sw}_D.log
timeout 900 python tools/sweep_rows_time.py D 10000 8 32 > gpurun_out/${1:-sw}_D8.log 2>&1; cat gpurun_out/${1:-sw}_D8.log

bash tools/r02_gpu.sh sw1 tests/test_gpu_sweep_rows.py tests/test_gpu_nccl_plumbing.py
timeout 600 python tools/sweep_rows_time.py C - 4 16 > gpurun_out/sw1_C.log 2>&1; cat gpurun_out/sw1_C.log
timeout 900 python tools/sweep_rows_time.py D - 8 32 > gpurun_out/sw1_D.log 2>&1; cat gpurun_out/sw1_D.log
timeout 900 python tools/sweep_rows_time.py D 10000 8 32 > gpurun_out/sw1_D8.log 2>&1; cat gpurun_out/sw1_D8.log

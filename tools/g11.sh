for r in 4 8 4 8; do MVN_K1_RPT=$r timeout 300 python tools/k1_time.py D 2>&1 | tail -1; done
MVN_K1_RPT=4 timeout 300 python tools/k1_time.py E 2>&1 | tail -1
bash tools/r02_gpu.sh g11 tests/test_gpu_potrf_dist.py tests/test_gpu_parity.py -k "not slow and not full_config and not max_size"

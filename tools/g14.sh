for rep in 1 2; do for lag in 0 1 3 8; do MVN_SOV_OZ_LAG=$lag timeout 600 python tools/sov_oz_time.py D 2 2>&1 | tail -1; done; done
MVN_SOV_OZ_LAG=3 timeout 300 python -m pytest tests/test_gpu_sov_int8.py -q -x 2>&1 | tail -1

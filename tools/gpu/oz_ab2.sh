timeout 600 python -m pytest tests/test_gpu_sov_int8.py -q -x 2>&1 | tail -1
for c in C D; do timeout 900 python tools/sov_oz_time.py $c 2 2>&1 | tail -1; done
timeout 900 python tools/sov_oz_check.py small 2>&1 | tail -5

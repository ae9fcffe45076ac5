for rep in 1 2; do MVN_K1_VARIANT=0 timeout 300 python tools/k1_time.py D 2>&1 | tail -1; done
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "matern" 2>&1 | tail -1
for c in A B C; do for s in 0 40 80 160 100000; do MVN_SOV_SERIAL=$s timeout 300 python tools/sov_time.py $c 3 2>&1 | tail -1; done; done
for s in 0 80; do MVN_SOV_SERIAL=$s timeout 300 python tools/sov_time.py D 1 2>&1 | tail -1; done

for rep in 1 2; do for v in 0 1 2 3 4; do MVN_K1_VARIANT=$v timeout 300 python tools/k1_time.py D 2>&1 | tail -1; done; done

#!/bin/bash
# A/B of the SOV GEMM warp count (compile-time MVN_SOV_GW): 8 (default) vs 16.
for gw in 8 16; do
  MVN_NVCC_EXTRA=-DMVN_SOV_GW=$gw python paper_2405_14892_b200/_build.py --force > /dev/null 2>&1
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m "gpu and not slow" -k "sov" 2>&1 | tail -1 | sed "s/^/gw=$gw tests: /"
  for c in B C D; do timeout 600 python tools/sov_time.py $c 2 2>&1 | tail -1 | sed "s/^/gw=$gw /"; done
done
python paper_2405_14892_b200/_build.py --force > /dev/null 2>&1

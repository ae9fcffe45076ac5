#!/bin/bash
# A/B of the SOV pipeline granularity (compile-time MVN_SOV_BK): 16 x 4 stages (default) vs 8 x 8.
for bk in 16 8; do
  MVN_NVCC_EXTRA=-DMVN_SOV_BK=$bk python paper_2405_14892_b200/_build.py --force > /dev/null 2>&1
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x -m "gpu and not slow" -k "sov" 2>&1 | tail -1 | sed "s/^/bk=$bk tests: /"
  for c in B C D; do timeout 600 python tools/sov_time.py $c 2 2>&1 | tail -1 | sed "s/^/bk=$bk /"; done
done
python paper_2405_14892_b200/_build.py --force > /dev/null 2>&1

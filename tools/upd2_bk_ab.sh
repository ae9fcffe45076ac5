#!/bin/bash
# A/B of the POTRF trailing-update ring granularity (compile-time MVN_UPD2_BK): 8 x 4 stages vs
# 16 x 2 (same bytes in flight, half the handshakes), alternating builds on one box.
mkdir -p gpurun_out/ub
for bk in 8 16; do
  MVN_NVCC_EXTRA="-DMVN_UPD2_BK=$bk" python paper_2405_14892_b200/_build.py --force > /dev/null 2>&1
  cp paper_2405_14892_b200/libmvn.so gpurun_out/ub/libmvn_bk$bk.so
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_potrf_dist.py -q -x -m "gpu and not slow" -k "potrf or update or panel" 2>&1 | tail -1 | sed "s/^/bk=$bk tests: /"
done
for rep in 1 2; do
  for bk in 8 16; do
    cp gpurun_out/ub/libmvn_bk$bk.so paper_2405_14892_b200/libmvn.so
    for c in D E; do timeout 600 python tools/potrf_time.py $c 2>&1 | tail -1 | sed "s/^/rep=$rep bk=$bk /"; done
  done
done
rm -rf gpurun_out/ub

#!/bin/bash
# A/B of the SOV pipeline granularity at D (compile-time MVN_SOV_BK): 32 x 2 stages vs 16 x 4,
# alternating builds on one box (the same bytes in flight; half the ring handshakes per flop).
mkdir -p gpurun_out/bk
for bk in 32 16; do
  MVN_NVCC_EXTRA=-DMVN_SOV_BK=$bk python paper_2405_14892_b200/_build.py --force > /dev/null 2>&1
  cp paper_2405_14892_b200/libmvn.so gpurun_out/bk/libmvn_bk$bk.so
done
for rep in 1 2 3; do
  for bk in 16 32; do
    cp gpurun_out/bk/libmvn_bk$bk.so paper_2405_14892_b200/libmvn.so
    for c in D; do timeout 600 python tools/sov_time.py $c 2 2>&1 | tail -1 | sed "s/^/rep=$rep bk=$bk /"; done
  done
done
for bk in 16 32; do
  cp gpurun_out/bk/libmvn_bk$bk.so paper_2405_14892_b200/libmvn.so
  for c in B E; do timeout 900 python tools/sov_time.py $c 1 2>&1 | tail -1 | sed "s/^/bk=$bk /"; done
done
rm -rf gpurun_out/bk

#!/bin/bash
# Headroom experiment: SOV with the Phi / Phi^-1 step replaced by a trivial one (MVN_SOV_FAKECHAIN,
# results wrong, timing only) vs the real chain.
for v in real fake; do
  if [ $v = fake ]; then MVN_NVCC_EXTRA=-DMVN_SOV_FAKECHAIN python paper_2405_14892_b200/_build.py --force > /dev/null 2>&1; fi
  for c in B C D; do timeout 600 python tools/sov_time.py $c 2 2>&1 | tail -1 | sed "s/^/$v /"; done
done
python paper_2405_14892_b200/_build.py --force > /dev/null 2>&1

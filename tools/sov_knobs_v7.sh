#!/bin/bash
# SOV producer knobs re-checked with the 32 x 2 ring at D (lag 0/2, hints 0/1), alternating.
for rep in 1 2; do
  for cfg in "0 1" "0 0" "2 1"; do
    set -- $cfg
    MVN_SOV_LAG=$1 MVN_SOV_HINTS=$2 timeout 600 python tools/sov_time.py D 2 2>&1 | tail -1 | sed "s/^/rep=$rep /"
  done
done

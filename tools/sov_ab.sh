#!/bin/bash
# A/B of the SOV producer knobs on one GPU. Usage: bash tools/sov_ab.sh TAG "C D"
TAG=${1:-ab}; CFGS=${2:-"C"}
for c in $CFGS; do
  for cfg in "0 0" "0 1" "2 1" "4 1" "1 1"; do
    set -- $cfg
    MVN_SOV_LAG=$1 MVN_SOV_HINTS=$2 timeout 600 python tools/sov_time.py $c 2 2>&1 | tail -1
  done
done

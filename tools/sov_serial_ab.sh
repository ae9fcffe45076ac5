#!/bin/bash
# A/B of MVN_SOV_SERIAL (row blocks whose GEMM waits for the previous chain). Usage: bash tools/sov_serial_ab.sh "B C D"
for c in ${1:-"C"}; do for v in 0 32 64 128 256; do MVN_SOV_SERIAL=$v timeout 600 python tools/sov_time.py $c 2 2>&1 | tail -1 | sed "s/^/serial=$v /"; done; done

#!/bin/bash
# Round-2 GPU check (run under gpurun, 1 GPU). Usage: bash tools/r02_gpu.sh TAG [tests...]
# Writes gpurun_out/TAG_*.log; prints a summary.
TAG=${1:-r02}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 300 python __graft_entry__.py --smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
if [ $# -gt 0 ]; then
  timeout 3000 python -m pytest "$@" -q -s -m gpu --durations=15 > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"
  grep -E "passed|failed|^E |config .:|s call|Error" gpurun_out/${TAG}_tests.log | tail -40
fi

#!/bin/bash
# Round profiling (run under gpurun, 1 GPU):
#   1. plain bench run (must exit 0 first), 2. ncu launch list of one bench step with per-launch
#   time and DRAM bytes (the `traffic` figure of bench.py's roofline), 3. optional full captures.
# Usage: bash tools/profile.sh TAG [CONFIG] [full]
TAG=${1:-r01}; CFG=${2:-D}; FULL=${3:-}
CMD="python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_${CFG}_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${CFG}_$TAG.csv $CMD > gpurun_out/ncu_launch_${CFG}_$TAG.log 2>&1
echo "launch list rc=$?"
if [ -n "$FULL" ]; then
  ncu --set full --clock-control none --import-source on -k regex:k_sov -c 1 -o gpurun_out/prof_sov_${CFG}_$TAG $CMD > gpurun_out/ncu_sov_${CFG}_$TAG.log 2>&1
  echo "sov full rc=$?"
fi

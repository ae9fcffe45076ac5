#!/bin/bash
# Launch list (bench config D, 1 step) + ncu --set full captures of the top kernels (config C).
# Usage under gpurun: bash tools/profile.sh <tag>
TAG=${1:-r01}
set -o pipefail
CMD_D="python bench.py --config D --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
CMD_C="python bench.py --config C --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
$CMD_D > gpurun_out/plain_D_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_D_$TAG.csv $CMD_D > gpurun_out/ncu_launch_D_$TAG.log 2>&1
echo "launch list rc=$?"
$CMD_C > gpurun_out/plain_C_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sov -c 1 -o gpurun_out/prof_sov_C_$TAG $CMD_C > gpurun_out/ncu_sov_C_$TAG.log 2>&1
echo "sov full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_update -s 20 -c 1 -o gpurun_out/prof_upd_C_$TAG $CMD_C > gpurun_out/ncu_upd_C_$TAG.log 2>&1
echo "update full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_potrf_diag|k_trsm|k_cov" -s 20 -c 3 -o gpurun_out/prof_misc_C_$TAG $CMD_C > gpurun_out/ncu_misc_C_$TAG.log 2>&1
echo "misc full rc=$?"

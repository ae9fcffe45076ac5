#!/bin/bash
# Full round check on one GPU (run under gpurun): smoke, all -m gpu tests, default bench line,
# ncu launch list of one bench step, ncu --set full captures of k_sov and k_update2.
# Usage: bash tools/round_gpu.sh TAG [CONFIG] [skip-tests]
TAG=${1:-r01}; CFG=${2:-D}; SKIP=${3:-}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/nvsmi_$TAG.txt 2>&1
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
if [ -z "$SKIP" ]; then
  timeout 1500 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/gpu_tests_$TAG.log
fi
timeout 900 python bench.py --config $CFG > gpurun_out/bench_${CFG}_$TAG.json 2> gpurun_out/bench_${CFG}_$TAG.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_${CFG}_$TAG.json
CMD="python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${CFG}_$TAG.csv $CMD > gpurun_out/ncu_launch_${CFG}_$TAG.log 2>&1
echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sov -c 1 -o gpurun_out/prof_sov_${CFG}_$TAG -f $CMD > gpurun_out/ncu_sov_${CFG}_$TAG.log 2>&1
echo "sov full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update2 -s 200 -c 1 -o gpurun_out/prof_upd_${CFG}_$TAG -f $CMD > gpurun_out/ncu_upd_${CFG}_$TAG.log 2>&1
echo "update full rc=$?"

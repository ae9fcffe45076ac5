#!/bin/bash
# End-of-round GPU check: smoke, every -m gpu test, the default bench line, the ncu launch list of
# the same command (per-launch times + DRAM bytes), and a config-E line.
TAG=${1:-r01v6}
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 2400 python -m pytest tests -q -m gpu --durations=8 > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|^E " gpurun_out/gpu_tests_$TAG.log | tail -8
timeout 900 python bench.py > gpurun_out/bench_D_$TAG.json 2> gpurun_out/bench_D_$TAG.err; echo "bench D rc=$?"
CMD="python bench.py --config D --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_D_$TAG.csv $CMD > gpurun_out/ncu_launch_D_$TAG.log 2>&1; echo "launch list rc=$?"
timeout 1500 python bench.py --config E --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_E_$TAG.json 2> gpurun_out/bench_E_$TAG.err; echo "bench E rc=$?"

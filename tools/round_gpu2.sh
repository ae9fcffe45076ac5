#!/bin/bash
# Round re-check after kernel changes (1 GPU): smoke, all -m gpu tests, default bench line, ncu launch
# list of one bench step, full ncu captures of k_update2 (one launch) and k_sov at a D-like reduced
# size (n = 32,761, N R = 20,000: ~0.6 s per replay). Usage: bash tools/round_gpu2.sh TAG
TAG=${1:-r01d}
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|^E " gpurun_out/gpu_tests_$TAG.log | tail -8
timeout 900 python bench.py > gpurun_out/bench_D_$TAG.json 2> gpurun_out/bench_D_$TAG.err; echo "bench rc=$?"; tail -c 2500 gpurun_out/bench_D_$TAG.json
CMD="python bench.py --config D --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_D_$TAG.csv $CMD > gpurun_out/ncu_launch_D_$TAG.log 2>&1; echo "launch list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update2 -s 60 -c 1 -o gpurun_out/prof_upd_D_$TAG -f $CMD > gpurun_out/ncu_upd_D_$TAG.log 2>&1; echo "update full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sov -c 1 -o gpurun_out/prof_sov_D181_$TAG -f python tools/sov_time.py D 0 181 20000 > gpurun_out/ncu_sov_D181_$TAG.log 2>&1; echo "sov D181 full rc=$?"

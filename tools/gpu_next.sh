#!/bin/bash
# NEXT-1/NEXT-2 checks + k_sov full capture at config C (run under gpurun, 1 GPU).
TAG=${1:-r01c}
timeout 900 python -m pytest tests/test_gpu_potrf_dist.py tests/test_gpu_mc.py -x -q -m gpu --durations=10 > gpurun_out/gpu_next_$TAG.log 2>&1; echo "next tests rc=$?"; tail -15 gpurun_out/gpu_next_$TAG.log
timeout 600 python bench.py --workload mc --config D --steps 3 --warmup 1 > gpurun_out/bench_mc_D_$TAG.json 2> gpurun_out/bench_mc_D_$TAG.err; echo "mc bench rc=$?"; tail -c 2500 gpurun_out/bench_mc_D_$TAG.json; tail -5 gpurun_out/bench_mc_D_$TAG.err
CMD="python bench.py --config C --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sov -c 1 -o gpurun_out/prof_sov_C_$TAG -f $CMD > gpurun_out/ncu_sov_C_$TAG.log 2>&1
echo "sov C full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mc_trmm -c 1 -o gpurun_out/prof_mc_C_$TAG -f python bench.py --workload mc --config C --steps 1 --warmup 0 --mc-samples 20000 > gpurun_out/ncu_mc_C_$TAG.log 2>&1
echo "mc C full rc=$?"

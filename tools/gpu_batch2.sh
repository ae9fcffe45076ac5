#!/bin/bash
# Parity of the new paths + POTRF super-panel A/B (run under gpurun, 1 GPU).
timeout 1200 python -m pytest tests/test_gpu_potrf_dist.py tests/test_gpu_posterior.py tests/test_gpu_parity.py tests/test_gpu_mc.py -q -m "gpu and not slow" > gpurun_out/t_b2.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/t_b2.log | tail -15
for c in C D; do for kp in 1 2 3; do MVN_POTRF_KP=$kp timeout 600 python tools/potrf_time.py $c 2 2>&1 | tail -1; done; done

#!/bin/bash
# Parity tests + quick benches on one GPU (used with gpurun). Usage: bash tools/gpu_check.sh TAG [configs...]
TAG=${1:-x}; shift
CFGS=${@:-"D"}
python __graft_entry__.py --smoke > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python -m pytest tests -x -q -m "gpu and not slow" > gpurun_out/gpu_tests_$TAG.log 2>&1; tail -3 gpurun_out/gpu_tests_$TAG.log
for c in $CFGS; do
  timeout 900 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_$TAG.log 2>&1
  python - "$c" "$TAG" <<'PY'
import json, sys
c, tag = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/bench_{c}_{tag}.log").read().strip().splitlines()[-1])
    print(c, "step_ms=%.1f" % d["ms_per_step"], "sov=%.1f ms frac=%.3f" % (d["stage_ms"]["sov"], d["roofline"]["frac"]),
          "potrf=%.1f ms %.2f TF" % (d["stage_ms"]["potrf"], d["cholesky_tflops"]), "clk", d["clocks"]["sm_mhz"])
except Exception as e:
    print(c, "FAILED", e); print(open(f"gpurun_out/bench_{c}_{tag}.log").read()[-2000:])
PY
done

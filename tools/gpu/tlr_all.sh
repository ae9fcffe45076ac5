# NEXT-3: TLR compression + TLR Cholesky GPU tests, then the 40K timings (both orders) and the
# compression-only line
TAG=${1:-ta}
timeout 1200 python -m pytest tests/test_gpu_tlr.py tests/test_gpu_tlr_potrf.py -q -m gpu --durations=8 > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|^E |FAILED" gpurun_out/${TAG}_tests.log | head -30
for ord in sorted spatial; do
  timeout 900 python bench.py --workload tlr-potrf --tlr-order $ord --steps 2 --warmup 1 > gpurun_out/${TAG}_${ord}.json 2> gpurun_out/${TAG}_${ord}.err; echo "bench $ord rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/${TAG}_${ord}.json').read().splitlines()[-1]);print({k:d[k] for k in ['value','dense_potrf_ms','tlr_over_dense','ranks_L','ranks_sigma','update_flops_over_dense_potrf','info','sov_on_Ltilde']}, d['roofline']['achieved'])" || tail -5 gpurun_out/${TAG}_${ord}.err
done
timeout 900 python bench.py --workload tlr --steps 2 --warmup 1 > gpurun_out/${TAG}_compress.json 2> gpurun_out/${TAG}_compress.err; echo "bench compress rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/${TAG}_compress.json').read().splitlines()[-1]);print(d['value'], d['ranks'], d['potrf_info_after'])"

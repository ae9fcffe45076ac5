# round-2 evidence: int8 public-call test, the int8 bench line (with e2e), ncu full captures
timeout 900 python -m pytest tests/test_gpu_sov_int8.py -q -x -k "mvn_crd" 2>&1 | tail -1
timeout 1200 python bench.py --sov-method 1 --potrf-method 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/p_bench_int8.json 2> gpurun_out/p_bench_int8.err; echo "bench int8 rc=$?"; python -c "import json;d=json.load(open('gpurun_out/p_bench_int8.json'));print(d['value'],d['stage_ms'],d['roofline']['frac'],d['clocks'],d['k_star'],d['e2e'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sov_oz -c 1 -o gpurun_out/p_sov_oz_D -f python tools/sov_oz_time.py D 0 > gpurun_out/p_ncu1.log 2>&1; echo "ncu sov_oz rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_upd_oz -s 10 -c 1 -o gpurun_out/p_upd_oz_D -f python tools/potrf_time.py D 1 - 1 > gpurun_out/p_ncu2.log 2>&1; echo "ncu upd_oz rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sov -c 1 -o gpurun_out/p_sov_C -f python tools/sov_time.py C 0 > gpurun_out/p_ncu3.log 2>&1; echo "ncu sov C rc=$?"

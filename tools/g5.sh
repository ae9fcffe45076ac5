timeout 120 python tools/sov_oz_check.py small > gpurun_out/g5_small.log 2>&1; echo "small rc=$?"; tail -8 gpurun_out/g5_small.log
timeout 300 python tools/sov_oz_check.py mid > gpurun_out/g5_mid.log 2>&1; echo "mid rc=$?"; tail -5 gpurun_out/g5_mid.log
bash tools/r02_gpu.sh g5 tests/test_gpu_potrf_dist.py -k "not super_panel_widths"
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g5_bench.json 2> gpurun_out/g5_bench.err; echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/g5_bench.json'));print(d['value'],d['stage_ms'],d['roofline']['frac'])"

bash tools/r02_gpu.sh g9 tests/test_gpu_potrf_int8.py tests/test_gpu_parity.py -k "potrf or matern or pack"
for m in 0 1; do timeout 600 python tools/potrf_time.py D 2 - $m 2>&1 | tail -1; done
timeout 600 python tools/potrf_time.py C 2 - 1 2>&1 | tail -1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g9_bench.json 2> gpurun_out/g9_bench.err; echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/g9_bench.json'));print(d['value'],d['stage_ms'],d['roofline']['frac'])"
for sr in 0 60 120; do MVN_SOV_SERIAL=$sr timeout 600 python bench.py --workload shard --config D --shard 8 --steps 2 --warmup 1 > gpurun_out/g9_shard_s$sr.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/g9_shard_s$sr.json'))
for w,v in d['shards'].items(): print('serial=$sr', w, round(v['sov_ms'],1), round(v['frac'],4))"; done

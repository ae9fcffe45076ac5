# end-of-round check on one GPU: smoke, the whole -m gpu suite, the driver's bench command, the
# mixed-precision line, the N > 1 code path on a one-rank communicator
TAG=${1:-final}
bash tools/r02_gpu.sh $TAG tests
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/${TAG}_bench.json').read().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['stage_ms'],d['roofline']['frac'],d['e2e']['value'],d['cpu_baseline']['value'],d['clocks'],d['k_star'])"
timeout 1500 python bench.py --sov-method 1 --potrf-method 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_int8.json 2> gpurun_out/${TAG}_bench_int8.err; echo "bench int8 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/${TAG}_bench_int8.json').read().splitlines()[-1]);print(d['value'],d['stage_ms'],d['roofline']['frac'],d['e2e']['value'],d['clocks'],d['k_star'])"
bash tools/gpu/multi_path.sh

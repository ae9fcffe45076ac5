# k_reduce_blocks rewrite (parallel ordered combine): the whole -m gpu suite, the small configs,
# a short D line and the launch list at A
TAG=${1:-rd}
timeout 2400 python -m pytest tests -q -m gpu -x --durations=5 > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_tests.log
bash tools/gpu/small_cfgs.sh $TAG
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_D.json 2> gpurun_out/${TAG}_D.err; echo "D rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/${TAG}_D.json').read().splitlines()[-1]);print(d['value'],d['stage_ms'],d['roofline']['frac'],d['k_star'])"
CMD="python bench.py --config A --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_A.csv $CMD > /dev/null 2>&1; echo "ncu A rc=$?"
CMD="python bench.py --config D --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_reduce_blocks --csv --log-file gpurun_out/${TAG}_launches_D_reduce.csv $CMD > /dev/null 2>&1; echo "ncu D rc=$?"

# per-config bench lines A, B, C (fp64 default path), no CPU baseline
TAG=${1:-sc}
for c in A B C; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_${c}.json 2> gpurun_out/${TAG}_${c}.err; echo "cfg $c rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/${TAG}_${c}.json').read().splitlines()[-1]);st=d['stage_ms'];print('$c', round(d['value']/1e9,3),'G', round(d['ms_per_step'],2),'ms', {k:round(v,3) for k,v in st.items()}, 'sov frac', round(d['roofline']['frac'],3), 'chol TF', round(d.get('cholesky_tflops',0),2))"
done

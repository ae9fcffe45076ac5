bash tools/r02_gpu.sh g3 tests/test_gpu_edges.py tests/test_gpu_parity.py -k "not slow and not full_config and not max_size"
for c in C D; do timeout 900 python bench.py --workload shard --config $c --shard 1,2,4,8 --steps 2 --warmup 1 > gpurun_out/g3_shard_$c.json 2>&1; echo "shard $c rc=$?"; python -c "
import json;d=json.load(open('gpurun_out/g3_shard_$c.json'))
for w,v in d['shards'].items(): print('$c', w, round(v['sov_ms'],1), round(v['frac'],4), v['widest_block'])"; done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g3_bench.json 2> gpurun_out/g3_bench.err; echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/g3_bench.json'));print(d['value'],d['stage_ms'],d['roofline']['frac'])"
# int8 MC method-2 ring depth experiment (bytes in flight per CTA), config D, 50,000 draws
for st in 3 2; do
  MVN_NVCC_EXTRA="-DMVN_OZ2_STAGES=$st" python paper_2405_14892_b200/_build.py --force > /dev/null 2>&1
  timeout 600 python bench.py --workload mc --mc-method 2 --config D --steps 3 --warmup 1 > gpurun_out/g3_mc2_st$st.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/g3_mc2_st$st.json'));print('stages=$st', d['ms_per_step'], d['roofline']['fp64_equivalent_tflops'], d['clocks'])"
done
python paper_2405_14892_b200/_build.py --force > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cov_matern -c 1 -o gpurun_out/g3_matern -f python bench.py --config D --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/g3_ncu.log 2>&1; echo "ncu rc=$?"

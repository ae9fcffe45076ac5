# per-rank shard efficiency vs the soft grid lockstep of the L panel (MVN_SOV_LAG), D and C at W = 8,
# plus the DRAM bytes of one W = 8 sweep at D
TAG=${1:-sl}
for cfg in D C; do
  for lag in 0 1 2 4; do
    MVN_SOV_LAG=$lag timeout 600 python bench.py --workload shard --config $cfg --shard 8 --steps 3 --warmup 1 > gpurun_out/${TAG}_${cfg}_${lag}.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/${TAG}_${cfg}_${lag}.json').read().splitlines()[-1]);s=d['shards']['8'];print('$cfg lag=$lag', round(s['sov_ms'],1), round(s['frac'],4), d['clocks'].get('sm_mhz'))"
  done
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_sov --csv --log-file gpurun_out/${TAG}_D8.csv python bench.py --workload shard --config D --shard 8 --steps 1 --warmup 0 > /dev/null 2>&1; echo "ncu rc=$?"
grep -E "k_sov" gpurun_out/${TAG}_D8.csv | awk -F'","' '{print $(NF-3), $(NF-2), $NF}' | head -12

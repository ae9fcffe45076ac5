# session-2 evidence: the launch list of one default bench step at D (per-kernel time + DRAM bytes),
# full ncu captures of the round-2 panel kernels (K2 / K3) and of the TLR kernels at n = 10,000
TAG=${1:-fe}
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches_D.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_launches.log 2>&1; echo "launch list rc=$?"
python tools/summarize_launches.py gpurun_out/${TAG}_launches_D.csv "one default bench step at D (fp64), session 2" | head -16
bash tools/gpu/diag_ncu.sh ${TAG}_dg
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tlr_compress|k_tlr_gemm" -s 100 -c 4 -o gpurun_out/${TAG}_tlr -f \
  python bench.py --workload tlr-potrf --tlr-g 100 --steps 1 --warmup 0 --tlr-sov-samples 2000 > gpurun_out/${TAG}_tlr_ncu.log 2>&1; echo "ncu tlr rc=$?"
for r in ${TAG}_dg ${TAG}_tlr; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active > gpurun_out/${r}_raw.csv 2>&1
  head -c 3000 gpurun_out/${r}_raw.csv | cut -c1-600; echo
done

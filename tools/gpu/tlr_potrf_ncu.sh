# NEXT-3 TLR Cholesky: ncu launch lists (per-kernel time shares) at n = 10,000 in both orders
TAG=${1:-tpn}
for ord in sorted spatial; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_${ord}.csv \
    python bench.py --workload tlr-potrf --tlr-order $ord --tlr-g 100 --steps 1 --warmup 0 > gpurun_out/${TAG}_${ord}_ncu.log 2>&1; echo "ncu $ord rc=$?"
  python tools/summarize_launches.py gpurun_out/${TAG}_${ord}.csv "TLR potrf n=10000 $ord" | head -20
done

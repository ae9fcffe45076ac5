# chain/GEMM contention A/B: MVN_SOV_SERIAL (the GEMM of row block rb waits for the chain of rb-1
# for rb * w <= serial * 128) on the small configs
for cfg in A B C; do
  for s in 0 40 200 100000; do
    MVN_SOV_SERIAL=$s timeout 600 python tools/sov_time.py $cfg 3
  done
done

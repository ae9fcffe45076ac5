set -x
nproc; lscpu | head -20; free -g | head -2; nvidia-smi
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 250 > gpurun_out/calib_clocks.csv &
SMI=$!
./tools/calib_fp64 > gpurun_out/calib_dmma.jsonl 2>&1
python tools/calib_fp64.py > gpurun_out/calib_dgemm.jsonl 2>&1
kill $SMI
cat gpurun_out/calib_dmma.jsonl gpurun_out/calib_dgemm.jsonl

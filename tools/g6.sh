timeout 600 python tools/sov_oz_check.py C,D > gpurun_out/g6_cd.log 2>&1; echo "cd rc=$?"; tail -4 gpurun_out/g6_cd.log
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader

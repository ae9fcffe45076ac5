# K1 (k_cov_matern) full ncu capture at config D: one launch
TAG=${1:-k1}
python tools/k1_time.py D > gpurun_out/${TAG}_time.log 2>&1 && cat gpurun_out/${TAG}_time.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cov_matern -s 2 -c 1 -o gpurun_out/${TAG} -f python tools/k1_time.py D > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/${TAG}_ncu.log

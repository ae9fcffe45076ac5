# small-n Cholesky latency + parity after a panel-kernel change
TAG=${1:-ps}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_potrf_dist.py tests/test_gpu_potrf_int8.py tests/test_gpu_edges.py -q -m gpu -x > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${TAG}_tests.log
python tools/potrf_small_time.py
python tools/potrf_time.py D 2
python tools/potrf_time.py B 5

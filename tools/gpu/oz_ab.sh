# int8 POTRF update + int8 SOV after the epilogue batching (tcgen05.ld x4 in flight, 16 global loads in flight)
for m in 1 0; do timeout 600 python tools/potrf_time.py D 2 - $m 2>&1 | tail -1; done
for c in C D; do timeout 900 python tools/sov_oz_time.py $c 2 2>&1 | tail -1; done
timeout 600 python -m pytest tests/test_gpu_potrf_int8.py tests/test_gpu_sov_int8.py -q -x 2>&1 | tail -1

bash tools/r02_gpu.sh g8 tests/test_gpu_sov_int8.py "tests/test_gpu_parity.py::test_full_config_all_samples_regions[E-1]"
timeout 900 python tools/sov_oz_check.py E > gpurun_out/g8_e.log 2>&1; echo "E rc=$?"; tail -2 gpurun_out/g8_e.log

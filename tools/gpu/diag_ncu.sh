# k_potrf_diag2 / k_trsm2 full ncu captures (source-level) at n = 4900
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_potrf_diag2|k_trsm2" -s 10 -c 2 -o gpurun_out/${1:-dg} -f python tools/potrf_small_time.py > gpurun_out/${1:-dg}_ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/${1:-dg}_ncu.log

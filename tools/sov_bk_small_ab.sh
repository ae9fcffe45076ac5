mkdir -p gpurun_out/ab
for bk in 16 32; do MVN_NVCC_EXTRA="-DMVN_SOV_BK=$bk" python paper_2405_14892_b200/_build.py --force > /dev/null 2>&1; cp paper_2405_14892_b200/libmvn.so gpurun_out/ab/l$bk.so; done
for rep in 1 2; do for bk in 16 32; do cp gpurun_out/ab/l$bk.so paper_2405_14892_b200/libmvn.so; for c in A B; do timeout 300 python tools/sov_time.py $c 5 2>&1 | tail -1 | sed "s/^/rep=$rep bk=$bk /"; done; done; done
for bk in 16 32; do cp gpurun_out/ab/l$bk.so paper_2405_14892_b200/libmvn.so; timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -1 | sed "s/^/bk=$bk /"; done
rm -rf gpurun_out/ab

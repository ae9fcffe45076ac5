#!/bin/bash
# NEXT-4 / NEXT-1 measurements, config E end to end, panel-SM A/B (1 GPU).
timeout 900 python bench.py --workload posterior --steps 3 --warmup 1 > gpurun_out/bench_post.json 2> gpurun_out/bench_post.err; echo "post rc=$?"; tail -c 1500 gpurun_out/bench_post.json; tail -3 gpurun_out/bench_post.err
timeout 900 python bench.py --workload potrf-dist --config D --steps 2 > gpurun_out/bench_pdist.json 2> gpurun_out/bench_pdist.err; echo "pdist rc=$?"; tail -c 1500 gpurun_out/bench_pdist.json; tail -3 gpurun_out/bench_pdist.err
for v in 4 6 8 12; do MVN_POTRF_PANEL_SMS=$v timeout 600 python tools/potrf_time.py D 2 2>&1 | tail -1 | sed "s/^/panel_sms=$v /"; done
timeout 1500 python bench.py --config E --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_E.json 2> gpurun_out/bench_E.err; echo "E rc=$?"; tail -c 2500 gpurun_out/bench_E.json; tail -3 gpurun_out/bench_E.err

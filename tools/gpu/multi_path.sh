# the N > 1 code path of bench.py on a one-rank NCCL communicator (collectives forced)
for extra in "" "--potrf dist" "--sov-method 1"; do
  NCCL_DEBUG=VERSION timeout 900 python bench.py --force-dist $extra --config C --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err; echo "force-dist [$extra] rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/m_bench.json').read().splitlines()[-1]);print(d['value'],d['potrf_mode'],d['config']['parallelism'],d['stage_ms_per_rank'] is not None,d['e2e']['api'],d['k_star'])" || tail -5 gpurun_out/m_bench.err
done
head -c 80 gpurun_out/m_bench.json; echo
# NEXT-1 on distributed storage end to end (one GPU: W = 1, and the forced NCCL path)
for extra in "" "--force-dist"; do
  timeout 900 python bench.py --potrf dstore $extra --config C --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/m_dstore.json 2> gpurun_out/m_dstore.err; echo "dstore [$extra] rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/m_dstore.json').read().splitlines()[-1]);print(d['value'],d['potrf_mode'],d['stage_ms'],d['e2e']['value'],d['gpu_launches'],d['k_star'])" || tail -5 gpurun_out/m_dstore.err
done

cd "$GRAFT_REPO_ROOT"
for c in c1 c4 c2; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
  tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), d['e2e']['d2h_bytes_per_step'])" || tail -5 gpurun_out/bench_$c.log
done
ARTEMIS_BENCH_SHARED_GPU=1 timeout 600 python bench.py --gpus 2 --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_2r.log 2> gpurun_out/bench_2r.err
tail -1 gpurun_out/bench_2r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('2 ranks shared', d['n_gpus'], round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3))" || tail -5 gpurun_out/bench_2r.err
timeout 300 python -m pytest tests/test_bench_contract.py -q -p no:cacheprovider -m gpu 2>&1 | tail -2

cd "$GRAFT_REPO_ROOT"
make -s -C oracle
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/cache_overhead.py > gpurun_out/cache_overhead.txt 2>&1; echo cache=$?; cat gpurun_out/cache_overhead.txt
for c in c2 c1 c4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
  tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), d['e2e']['d2h_bytes_per_step'], 'api', d.get('e2e_api') and round(d['e2e_api']['ms_per_step'],2), d.get('e2e_api') and round(d['e2e_api']['identity_policy']['ms_per_step'],2))"
done
bash scripts/gpu_exp3.sh | tail -9

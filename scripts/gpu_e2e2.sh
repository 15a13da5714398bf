cd "$GRAFT_REPO_ROOT"
make -s -C oracle
timeout 600 python scripts/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1; echo probe=$?
cat gpurun_out/e2e_probe.log | tail -12
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_e2e.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_e2e.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e_api']['ms_per_step'], d['e2e_api']['identity_policy']['ms_per_step'])"

cd "$GRAFT_REPO_ROOT"
make -s -C oracle
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke4.log 2>&1; echo smoke=$?
timeout 600 python -m pytest tests/test_fk_native.py -q -x > gpurun_out/pytest_fk.log 2>&1; echo fk=$?; tail -1 gpurun_out/pytest_fk.log
timeout 600 python scripts/e2e_probe.py > gpurun_out/e2e_probe4.log 2>&1; echo probe=$?
tail -8 gpurun_out/e2e_probe4.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_e2e4.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_e2e4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e_api']['ms_per_step'], d['e2e_api']['identity_policy']['ms_per_step'])"
for c in c1 c4; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo $c=$?; tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_step'])"; done

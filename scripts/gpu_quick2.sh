set -x
cd "$GRAFT_REPO_ROOT"
make -s -C oracle
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$?
tail -5 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/frame', d['ms_per_step'], 'e2e', d['e2e'], 'stages', d['stage_ms'], 'frac', d['roofline']['frac'])"

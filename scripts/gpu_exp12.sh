cd "$GRAFT_REPO_ROOT"
make -s -C oracle
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "configs or edges or races or pipeline" > gpurun_out/pytest_views.log 2>&1
echo pytest=$?; tail -2 gpurun_out/pytest_views.log
bash scripts/gpu_quick.sh
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 bench', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'])"

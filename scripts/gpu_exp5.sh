cd "$GRAFT_REPO_ROOT"
make -s -C oracle
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
bash scripts/gpu_exp3.sh | tail -10
for i in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stage_ms']; print(round(d['ms_per_step'],4), {k: round(v,4) for k,v in s.items()})"
done

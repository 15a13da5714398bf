# quick same-box timing: bench c2 x2 + configs c4 c1 c0
cd "$GRAFT_REPO_ROOT"
for i in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stage_ms']; print(round(d['ms_per_step'],4), {k: round(v,4) for k,v in s.items()})"
done
timeout 900 python scripts/bench_configs.py c4 c1 c0 2>/dev/null | python -c "import sys,json; print(' '.join(json.loads(l)['config']+'='+str(round(json.loads(l)['ms_per_step'],3)) for l in sys.stdin))"

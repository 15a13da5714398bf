# same-box A/B of an environment switch: scripts/gpu_ab_env.sh VAR  (VAR=1 vs VAR=0)
cd "$GRAFT_REPO_ROOT"
V=${1:-ARTEMIS_PDL}
for r in 1 2; do
  for val in 1 0; do
    c2=$(env $V=$val timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stage_ms']; print(round(d['ms_per_step'],4), round(s['render'],4))")
    cf=$(env $V=$val timeout 900 python scripts/bench_configs.py c4 c1 c0 2>/dev/null | python -c "import sys,json; print(' '.join(json.loads(l)['config']+'='+str(round(json.loads(l)['ms_per_step'],3)) for l in sys.stdin))")
    echo "$V=$val c2=$c2 $cf"
  done
done

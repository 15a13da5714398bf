cd "$GRAFT_REPO_ROOT"
for o in auto rowmajor centre auto; do
  if [ $o = auto ]; then unset ARTEMIS_TILE_ORDER; else export ARTEMIS_TILE_ORDER=$o; fi
  r=$(timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4))")
  c=$(timeout 600 python scripts/bench_configs.py c4 c1 c0 2>/dev/null | python -c "import sys,json; print(' '.join(json.loads(l)['config']+'='+str(round(json.loads(l)['ms_per_step'],3)) for l in sys.stdin))")
  echo "$o bench_c2 $r $c"
done
unset ARTEMIS_TILE_ORDER
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2

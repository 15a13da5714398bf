# experiment: streaming output stores / L2 evict_last row hint / render grid caps (c4)
cd "$GRAFT_REPO_ROOT"
python scripts/build_variants.py sout rhint sout_rhint > /dev/null 2>&1
VARIANTS="base sout rhint sout_rhint" bash scripts/gpu_var_sweep.sh
for cap in 444 296 148; do
  c=$(ARTEMIS_RENDER_BLOCKS=$cap timeout 900 python scripts/bench_configs.py c4 2>/dev/null | python -c "import sys,json; print(' '.join(json.loads(l)['config']+'='+str(round(json.loads(l)['ms_per_step'],3)) for l in sys.stdin))")
  echo "cap $cap $c"
done

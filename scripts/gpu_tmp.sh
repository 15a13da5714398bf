cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_edges.py tests/test_gpu_configs.py -q -x -p no:cacheprovider 2>&1 | tail -2
for m in 0 1; do
c=$(ARTEMIS_VIEWS_SEPARATE=$m timeout 900 python scripts/bench_configs.py c4 c1 2>/dev/null | python -c "import sys,json; print(' '.join(json.loads(l)['config']+'='+str(round(json.loads(l)['ms_per_step'],3)) for l in sys.stdin))")
echo "separate=$m $c"
done

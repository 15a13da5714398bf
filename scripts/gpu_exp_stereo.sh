cd "$GRAFT_REPO_ROOT"
run() { timeout 900 python scripts/bench_configs.py c4 2>/dev/null | python -c "import sys,json; print(' '.join(json.loads(l)['config']+'='+str(round(json.loads(l)['ms_per_step'],3)) for l in sys.stdin))"; }
echo "separate $(run)"
echo "one $(ARTEMIS_VIEWS_ONE_LAUNCH=1 run)"
for sh in "0,8" "0,-8" "0,4" "0,-4" "0,12" "0,-12"; do echo "one shift $sh $(ARTEMIS_VIEWS_ONE_LAUNCH=1 ARTEMIS_VIEW_SHIFT=$sh run)"; done
echo "separate $(run)"

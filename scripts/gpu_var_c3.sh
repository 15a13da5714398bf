cd "$GRAFT_REPO_ROOT"
for v in base t64 base t64; do
  if [ $v = base ]; then LP=$PWD/paper_2202_05628_b200/libartemis.so; else LP=$PWD/variants/libartemis_$v.so; fi
  c=$(ARTEMIS_LIB_PATH=$LP timeout 900 python scripts/bench_configs.py c3 c2 2>/dev/null | python -c "import sys,json; print(' '.join(json.loads(l)['config']+'='+str(round(json.loads(l)['ms_per_step'],3)) for l in sys.stdin))")
  echo "var $v $c"
done

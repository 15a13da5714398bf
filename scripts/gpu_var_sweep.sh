# Library-variant sweep: bench.py (configs[2]) plus configs[4] and configs[1] per variant:
#   VARIANTS="base x y" bash scripts/gpu_var_sweep.sh
cd "$GRAFT_REPO_ROOT"
for v in ${VARIANTS:-base}; do
  if [ $v = base ]; then LP=$PWD/paper_2202_05628_b200/libartemis.so; else LP=$PWD/variants/libartemis_$v.so; fi
  r=$(ARTEMIS_LIB_PATH=$LP timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4))")
  c=$(ARTEMIS_LIB_PATH=$LP timeout 900 python scripts/bench_configs.py c4 c1 2>/dev/null | python -c "import sys,json; print(' '.join(json.loads(l)['config']+'='+str(round(json.loads(l)['ms_per_step'],3)) for l in sys.stdin))")
  echo "var $v bench=$r $c"
done

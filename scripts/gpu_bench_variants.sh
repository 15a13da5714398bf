# bench.py device time (graph replay, L2 flushed) per library variant:
#   VARIANTS="base x y" bash scripts/gpu_bench_variants.sh
cd "$GRAFT_REPO_ROOT"
for v in ${VARIANTS:-base}; do
  if [ $v = base ]; then LP=$PWD/paper_2202_05628_b200/libartemis.so; else LP=$PWD/variants/libartemis_$v.so; fi
  ARTEMIS_LIB_PATH=$LP timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), 'render', round(d['stage_ms']['render'],4))"
done

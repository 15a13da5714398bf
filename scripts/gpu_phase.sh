cd "$GRAFT_REPO_ROOT"
ARTEMIS_LIB_PATH=$PWD/variants/libartemis_clocks.so timeout 300 python scripts/phase_clocks.py 2>&1 | tail -4
for v in base b5 b6; do
  if [ $v = base ]; then LP=$PWD/paper_2202_05628_b200/libartemis.so; else LP=$PWD/variants/libartemis_$v.so; fi
  ARTEMIS_LIB_PATH=$LP timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['stage_ms']['render'])"
done

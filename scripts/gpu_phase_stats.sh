cd "$GRAFT_REPO_ROOT"
python scripts/build_variants.py clocks noshade > /dev/null 2>&1
ARTEMIS_LIB_PATH=$PWD/variants/libartemis_clocks.so timeout 300 python scripts/phase_clocks.py 2>&1 | tail -4
for v in noshade; do
  ARTEMIS_LIB_PATH=$PWD/variants/libartemis_$v.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['stage_ms']['render'])"
done

cd "$GRAFT_REPO_ROOT"
for v in variants/libartemis_*.so; do
  n=$(basename $v .so)
  ARTEMIS_LIB_PATH=$PWD/$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sweep_$n.log 2>&1
  echo "$n $(tail -1 gpurun_out/sweep_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d['stage_ms']['render'],3))" 2>&1 | tail -1)"
done

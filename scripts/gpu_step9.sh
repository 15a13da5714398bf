cd "$GRAFT_REPO_ROOT"
make -s -C oracle
timeout 900 python -m pytest tests -m gpu -x -q -k "stream or pipeline or bench" > gpurun_out/pytest_step9.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_step9.log
for r in 1 2; do
  for mode in "ARTEMIS_STREAM_TWIN=1" "ARTEMIS_STREAM_TWIN=0"; do
    c2=$(env $mode timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4))")
    c0=$(env $mode timeout 300 python bench.py --config c0 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4))")
    echo "$mode c2=$c2 c0=$c0"
  done
done
timeout 600 python scripts/e2e_probe.py > gpurun_out/e2e_probe9.log 2>&1; tail -7 gpurun_out/e2e_probe9.log

cd "$GRAFT_REPO_ROOT"
make -s -C oracle
timeout 900 python -m pytest tests -m gpu -x -q -k "pipeline or edges or configs or peer or races or traces" > gpurun_out/pytest_step10.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_step10.log
timeout 600 python scripts/timeline.py c2 6 > gpurun_out/timeline10_c2.txt 2>&1; echo tl=$?
tail -12 gpurun_out/timeline10_c2.txt
for r in 1 2; do
  for mode in "ARTEMIS_CLEAR_FIRST=0" "ARTEMIS_CLEAR_FIRST=1"; do
    c2=$(env $mode timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stage_ms']; print(round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), d['gpu_launches'])")
    cf=$(env $mode timeout 900 python scripts/bench_configs.py c4 c1 c0 2>/dev/null | python -c "import sys,json; print(' '.join(json.loads(l)['config']+'='+str(round(json.loads(l)['ms_per_step'],3)) for l in sys.stdin))")
    echo "$mode c2=$c2 $cf"
  done
done

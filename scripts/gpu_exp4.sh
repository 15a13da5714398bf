cd "$GRAFT_REPO_ROOT"
make -s -C oracle
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "pipeline or traces or configs or races or edges" > gpurun_out/pytest_counting.log 2>&1
echo pytest=$?; tail -2 gpurun_out/pytest_counting.log
bash scripts/gpu_exp3.sh
for c in 1 0 1 0; do
  r=$(ARTEMIS_COUNTING=$c timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stage_ms']; print(round(d['ms_per_step'],4), {k: round(v,4) for k,v in s.items()})")
  echo "counting=$c $r"
done
c=$(timeout 900 python scripts/bench_configs.py c4 c1 c0 2>/dev/null | python -c "import sys,json; print(' '.join(json.loads(l)['config']+'='+str(round(json.loads(l)['ms_per_step'],3)) for l in sys.stdin))")
echo "counting=1 $c"
c=$(ARTEMIS_COUNTING=0 timeout 900 python scripts/bench_configs.py c4 c1 c0 2>/dev/null | python -c "import sys,json; print(' '.join(json.loads(l)['config']+'='+str(round(json.loads(l)['ms_per_step'],3)) for l in sys.stdin))")
echo "counting=0 $c"

cd "$GRAFT_REPO_ROOT"
make -s -C oracle
python scripts/div_selftest.py
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "traces or kernels or races or pipeline or configs or edges" > gpurun_out/pytest_fast.log 2>&1
echo pytest=$?; tail -2 gpurun_out/pytest_fast.log
for e in 1 0 1 0; do
  r=$(ARTEMIS_FAST_DIV=$e timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['stage_ms']['render'],4))")
  c=$(ARTEMIS_FAST_DIV=$e timeout 900 python scripts/bench_configs.py c4 c1 c0 2>/dev/null | python -c "import sys,json; print(' '.join(json.loads(l)['config']+'='+str(round(json.loads(l)['ms_per_step'],3)) for l in sys.stdin))")
  echo "fastdiv=$e c2=$r $c"
done

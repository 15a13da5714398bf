# same-box A/B of library variants: bench c2 + configs c4 c1, twice each
#   VARIANTS="base bpf" bash scripts/gpu_ab_variants.sh
cd "$GRAFT_REPO_ROOT"
for r in 1 2; do
  for v in ${VARIANTS:-base}; do
    if [ $v = base ]; then LP=$PWD/paper_2202_05628_b200/libartemis.so; else LP=$PWD/variants/libartemis_$v.so; fi
    c2=$(ARTEMIS_LIB_PATH=$LP timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stage_ms']; print(round(d['ms_per_step'],4), {k: round(x,4) for k,x in s.items()})")
    cf=$(ARTEMIS_LIB_PATH=$LP timeout 900 python scripts/bench_configs.py ${CONFIGS:-c4 c1} 2>/dev/null | python -c "import sys,json; print(' '.join(json.loads(l)['config']+'='+str(round(json.loads(l)['ms_per_step'],3)) for l in sys.stdin))")
    echo "$v c2=$c2 $cf"
  done
done

cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "pipeline or traces or races or edges" > gpurun_out/pytest_counting.log 2>&1
echo pytest=$?; tail -2 gpurun_out/pytest_counting.log
bash scripts/gpu_exp3.sh | tail -9
python scripts/build_variants.py q4b5 q4t40b5 q4t56b5 > /dev/null 2>&1
VARIANTS="base q4b5 q4t40b5 q4t56b5 base q4b5" bash scripts/gpu_var_sweep.sh

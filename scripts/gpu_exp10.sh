cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "traces or kernels or races or pipeline or configs" > gpurun_out/pytest_fast.log 2>&1
echo pytest=$?; tail -2 gpurun_out/pytest_fast.log
python scripts/build_variants.py slowcam norcp > /dev/null 2>&1
VARIANTS="base slowcam norcp base slowcam" bash scripts/gpu_var_sweep.sh

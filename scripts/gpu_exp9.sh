cd "$GRAFT_REPO_ROOT"
python scripts/build_variants.py rcp > /dev/null 2>&1
ARTEMIS_LIB_PATH=$PWD/variants/libartemis_rcp.so timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "traces or kernels or races or pipeline" > gpurun_out/pytest_rcp.log 2>&1
echo pytest_rcp=$?; tail -2 gpurun_out/pytest_rcp.log
VARIANTS="base rcp base rcp" bash scripts/gpu_var_sweep.sh

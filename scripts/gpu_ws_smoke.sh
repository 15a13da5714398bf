cd "$GRAFT_REPO_ROOT"
make -s -C oracle
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3; echo smoke=$?
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
VARIANTS="ws0" timeout 600 bash scripts/gpu_sweep2.sh

cd "$GRAFT_REPO_ROOT"
make -s -C oracle
timeout 900 python -m pytest tests -m gpu -x -q -k "pipeline or edges or configs or traces" > gpurun_out/pytest_step1.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_step1.log
VARIANTS="base bpf" bash scripts/gpu_ab_variants.sh

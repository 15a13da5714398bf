cd "$GRAFT_REPO_ROOT"
VARIANTS="base prev base prev" bash scripts/gpu_bench_variants.sh
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2

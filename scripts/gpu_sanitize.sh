# one compute-sanitizer tool per call: bash scripts/gpu_sanitize.sh <tool>
cd "$GRAFT_REPO_ROOT"
tool=${1:-memcheck}
timeout 300 python scripts/sanitize_target.py > gpurun_out/san_plain.log 2>&1 && \
timeout 2400 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
    python scripts/sanitize_target.py > gpurun_out/sanitize_$tool.log 2>&1
echo sanitize_$tool=$?
tail -15 gpurun_out/sanitize_$tool.log

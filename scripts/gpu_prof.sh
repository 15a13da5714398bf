set -x
cd "$GRAFT_REPO_ROOT"
timeout 300 python scripts/prof_frame.py c2 3 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 1 -c 1 \
    -o gpurun_out/prof_render python scripts/prof_frame.py c2 3 > gpurun_out/ncu_render.log 2>&1
echo ncu=$?

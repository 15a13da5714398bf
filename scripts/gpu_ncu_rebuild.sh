cd "$GRAFT_REPO_ROOT"
timeout 300 python scripts/prof_frame.py c2 2 > gpurun_out/plain_rb.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lbs_warp_kernel|build_tree_kernel" -s 2 -c 2 \
    -o gpurun_out/prof_rebuild python scripts/prof_frame.py c2 2 > gpurun_out/ncu_rb.log 2>&1
echo ncu=$?

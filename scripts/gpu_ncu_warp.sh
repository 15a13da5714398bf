cd "$GRAFT_REPO_ROOT"
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"lbs_warp_kernel" -s 2 -c 1 \
    -o gpurun_out/prof_warp python scripts/prof_frame.py c2 3 > gpurun_out/ncu_warp.log 2>&1
echo ncu_warp=$?

# ncu --set full of the rebuild kernels of one c2 frame (warp, slot, Karras build)
cd "$GRAFT_REPO_ROOT"
timeout 300 python scripts/prof_frame.py c2 3 > gpurun_out/prof_plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"lbs_warp_kernel|slot_kernel|build_tree32_kernel" -s 6 -c 3 \
    -o gpurun_out/prof_rebuild python scripts/prof_frame.py c2 3 > gpurun_out/ncu_rebuild.log 2>&1
echo ncu_rebuild=$?

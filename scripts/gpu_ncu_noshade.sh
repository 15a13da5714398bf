# ncu --set full of the no-shading render variant (traversal + integration only)
cd "$GRAFT_REPO_ROOT"
python scripts/build_variants.py noshade > /dev/null 2>&1
export ARTEMIS_LIB_PATH=$PWD/variants/libartemis_noshade.so
timeout 300 python scripts/prof_frame.py c2 2 > gpurun_out/plain_noshade.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 1 -c 1 \
    -o gpurun_out/prof_noshade python scripts/prof_frame.py c2 2 > gpurun_out/ncu_noshade.log 2>&1
echo ncu=$?

cd "$GRAFT_REPO_ROOT"
make -s -C oracle
timeout 900 python -m pytest tests -m gpu -x -q -k "pipeline or edges or kernels or configs" > gpurun_out/pytest_step3.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_step3.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none \
     -k regex:"lbs_warp|count_kernel|scan2|emit_kernel|slot_kernel|finish_kernel|build_tree" --csv --log-file gpurun_out/rb3.csv python scripts/prof_frame.py c2 3 > /dev/null 2>&1
python scripts/ncu_launch_table.py gpurun_out/rb3.csv 2>/dev/null | tail -7
CONFIGS="c4 c1 c0" VARIANTS="base" bash scripts/gpu_ab_variants.sh

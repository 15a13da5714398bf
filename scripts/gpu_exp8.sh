cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "pipeline or traces or races or edges or configs" > gpurun_out/pytest_counting.log 2>&1
echo pytest=$?; tail -2 gpurun_out/pytest_counting.log
bash scripts/gpu_exp3.sh | tail -10
bash scripts/gpu_quick.sh
timeout 600 python scripts/c4_rows.py > gpurun_out/c4_rows.json 2>&1; echo c4rows=$?; tail -1 gpurun_out/c4_rows.json
timeout 300 python scripts/prof_frame.py c4 1 > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -k regex:render_kernel --clock-control none --csv --log-file gpurun_out/c4_render.csv python scripts/prof_frame.py c4 1 > gpurun_out/ncu_c4.log 2>&1
echo c4ncu=$?; grep -E "dram__bytes_read|gpu__time" gpurun_out/c4_render.csv | cut -c1-300

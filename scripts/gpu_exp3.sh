cd "$GRAFT_REPO_ROOT"
timeout 300 python scripts/prof_frame.py c2 3 > gpurun_out/plain_cnt.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_cnt.csv python scripts/prof_frame.py c2 3 > gpurun_out/ncu_cnt.log 2>&1
echo launches=$?
python scripts/launch_list.py gpurun_out/launches_cnt.csv 2>&1 | tail -22

# counting rebuild kernel durations; flat-shade variant A/B; L2 traffic decomposition
cd "$GRAFT_REPO_ROOT"
python scripts/build_variants.py flat nopf > /dev/null 2>&1
timeout 300 python scripts/prof_frame.py c2 3 > gpurun_out/plain_cnt.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 40 --csv \
    --log-file gpurun_out/launches_cnt.csv python scripts/prof_frame.py c2 3 > gpurun_out/ncu_cnt.log 2>&1
echo launches=$?
python scripts/launch_list.py gpurun_out/launches_cnt.csv 2>/dev/null | tail -25
VARIANTS="base flat base flat" bash scripts/gpu_var_sweep.sh
bash scripts/gpu_l2_traffic.sh

set -x
cd "$GRAFT_REPO_ROOT"
timeout 300 python scripts/prof_frame.py c2 3 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s 20 --csv --log-file gpurun_out/launches.csv python scripts/prof_frame.py c2 3 > gpurun_out/ncu_launches.log 2>&1
echo launches=$?

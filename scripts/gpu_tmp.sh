cd "$GRAFT_REPO_ROOT"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:onesweep -s 5 -c 1 -o gpurun_out/prof_sort python scripts/prof_frame.py c2 2 > gpurun_out/ncu_sort.log 2>&1
echo rc=$?

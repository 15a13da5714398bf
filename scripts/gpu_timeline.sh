cd "$GRAFT_REPO_ROOT"
timeout 600 python scripts/timeline.py c2 6 > gpurun_out/timeline_c2.txt 2>&1; echo tl=$?
tail -45 gpurun_out/timeline_c2.txt

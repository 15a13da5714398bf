# Per-kernel HBM GB/s and L2 hit rate of one configs[2] frame (ncu, one GPU).
cd "$GRAFT_REPO_ROOT"
timeout 300 python scripts/prof_frame.py c2 3 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -s 20 --csv --log-file gpurun_out/kernels.csv python scripts/prof_frame.py c2 3 > gpurun_out/ncu_kernels.log 2>&1
echo kernels=$?

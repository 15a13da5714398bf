# Per-kernel table of the current build (c2 frame) + launch list of the bench.
cd "$GRAFT_REPO_ROOT"
bash scripts/gpu_kernel_table.sh
timeout 300 python scripts/prof_frame.py c4 2 > gpurun_out/prof_c4_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum \
    --clock-control none -s 9 --csv --log-file gpurun_out/kernels_c4.csv python scripts/prof_frame.py c4 2 > gpurun_out/ncu_kernels_c4.log 2>&1
echo c4=$?

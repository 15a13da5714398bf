# Round-2 final evidence on ONE GPU: smoke, bench (CPU baseline + e2e + e2e_api),
# reference arm, c1/c4 bench lines, all configs, per-kernel table, launch list
# of the bench command, render + rebuild ncu --set full, frame timeline.
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/lscpu.txt
make -s -C oracle
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo benchref=$?
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1; echo bench_c1=$?
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo bench_c4=$?
timeout 900 python scripts/bench_configs.py > gpurun_out/configs.jsonl 2>gpurun_out/configs.err; echo configs=$?
timeout 600 python scripts/timeline.py c2 6 > gpurun_out/timeline_c2.txt 2>&1; echo timeline=$?
timeout 300 python scripts/prof_frame.py c2 3 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -s 9 --csv --log-file gpurun_out/kernels.csv python scripts/prof_frame.py c2 3 > gpurun_out/ncu_kernels.log 2>&1
echo kernels=$?
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches.log 2>&1
echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 1 -c 1 \
    -o gpurun_out/prof_render python scripts/prof_frame.py c2 3 > gpurun_out/ncu_render.log 2>&1
echo ncu_render=$?
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"lbs_warp_kernel|slot_kernel|finish_kernel|build_tree32_kernel" -s 8 -c 4 \
    -o gpurun_out/prof_rebuild python scripts/prof_frame.py c2 3 > gpurun_out/ncu_rebuild.log 2>&1
echo ncu_rebuild=$?
tail -1 gpurun_out/bench.log | cut -c1-400

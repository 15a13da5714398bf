# same-box A/B of rebuild variants: per-kernel ncu durations (metrics only) + bench
cd "$GRAFT_REPO_ROOT"
for v in ${VARIANTS:-base}; do
  if [ $v = base ]; then LP=$PWD/paper_2202_05628_b200/libartemis.so; else LP=$PWD/variants/libartemis_$v.so; fi
  ARTEMIS_LIB_PATH=$LP timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none \
     -k regex:"lbs_warp|count_kernel|scan2|emit_kernel|slot_kernel|finish_kernel|build_tree" -s 16 --csv --log-file gpurun_out/rb_$v.csv python scripts/prof_frame.py c2 3 > /dev/null 2>&1
  python scripts/ncu_launch_table.py gpurun_out/rb_$v.csv 2>/dev/null | sed "s/^/$v /" || echo "$v failed"
done
bash scripts/gpu_ab_variants.sh

# Kernel durations (ncu, cold serialised) of one c2 frame per library variant:
#   VARIANTS="base e5" bash scripts/gpu_variant_times.sh
cd "$GRAFT_REPO_ROOT"
for v in ${VARIANTS:-base}; do
  if [ $v = base ]; then LP=$PWD/paper_2202_05628_b200/libartemis.so; else LP=$PWD/variants/libartemis_$v.so; fi
  ARTEMIS_LIB_PATH=$LP ARTEMIS_SHADE_BLOCKS_PER_SM=${SBPS:-0} timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum,l1tex__t_sector_hit_rate.pct --clock-control none \
     -k regex:"render_kernel|shade_kernel" -s 3 --csv --log-file gpurun_out/vt_$v.csv python scripts/prof_frame.py c2 2 > /dev/null 2>&1
  python scripts/ncu_launch_table.py gpurun_out/vt_$v.csv 2>/dev/null | sed "s/^/$v /" || echo "$v failed"
done

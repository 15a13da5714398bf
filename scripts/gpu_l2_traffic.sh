# L2 traffic decomposition of render_kernel (configs[2] frame): base vs no row prefetch
cd "$GRAFT_REPO_ROOT"
python scripts/build_variants.py nopf > /dev/null 2>&1
M=gpu__time_duration.sum,lts__t_bytes.sum,lts__t_sectors.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_requests_op_read.sum,lts__t_sectors_op_read_lookup_hit.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum,l1tex__t_bytes.sum,sm__inst_executed.sum
for v in base nopf; do
  if [ $v = base ]; then LP=$PWD/paper_2202_05628_b200/libartemis.so; else LP=$PWD/variants/libartemis_$v.so; fi
  ARTEMIS_LIB_PATH=$LP timeout 300 python scripts/prof_frame.py c2 2 > gpurun_out/plain_$v.log 2>&1 && \
  ARTEMIS_LIB_PATH=$LP timeout 600 ncu --metrics $M --clock-control none -k regex:render_kernel -s 1 -c 1 --csv \
      --log-file gpurun_out/l2_$v.csv python scripts/prof_frame.py c2 2 > gpurun_out/ncu_l2_$v.log 2>&1
  echo "$v ncu=$?"
  python - "$v" <<'PY'
import csv, sys
v = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/l2_{v}.csv")))
hdr = None
for r in rows:
    if "Metric Name" in r:
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r)); print(v, d["Metric Name"], d["Metric Unit"], d["Metric Value"])
PY
done

# Full round check on ONE GPU: smoke, gpu tests, bench (with CPU baseline and
# e2e), launch list and a full ncu capture of the render kernel.
set -x
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
make -s -C oracle
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo benchref=$?
tail -5 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench.log; tail -1 gpurun_out/bench_ref.log
if [ "${PROFILE:-1}" = "1" ]; then
  timeout 300 python scripts/prof_frame.py c2 3 > gpurun_out/prof_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -s 20 --csv --log-file gpurun_out/launches.csv python scripts/prof_frame.py c2 3 > gpurun_out/ncu_launches.log 2>&1
  echo launches=$?
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 1 -c 1 \
      -o gpurun_out/prof_render python scripts/prof_frame.py c2 3 > gpurun_out/ncu_render.log 2>&1
  echo ncu=$?
fi

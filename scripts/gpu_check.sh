set -x
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
make -s -C oracle
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$?
tail -5 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/bench.log
if [ "${PROFILE:-0}" = "1" ]; then
  timeout 300 python scripts/prof_frame.py c2 3 > gpurun_out/prof_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 1 -c 1 \
      -o gpurun_out/prof_render python scripts/prof_frame.py c2 3 > gpurun_out/ncu_render.log 2>&1
  echo ncu=$?
fi

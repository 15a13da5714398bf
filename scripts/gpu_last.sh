# Last check of the final build: smoke, full GPU suite, bench line (c2), reference arm.
cd "$GRAFT_REPO_ROOT"
make -s -C oracle
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_last.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_last.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_last.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_last.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_last.log 2>&1; echo benchref=$?
tail -1 gpurun_out/bench_last.log | cut -c1-300

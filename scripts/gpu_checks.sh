# Bounds-checking build (-DARTEMIS_DEBUG_CHECKS: shared-memory queue/stack,
# scatter and index asserts that trap) over the race/determinism tests and
# the parity suites -- in place of compute-sanitizer, which is closed on the
# GPU pool.
cd "$GRAFT_REPO_ROOT"
python scripts/build_variants.py checks > gpurun_out/checks_build.log 2>&1 || { echo build failed; tail -20 gpurun_out/checks_build.log; exit 1; }
ARTEMIS_LIB_PATH=$PWD/variants/libartemis_checks.so timeout 1800 python -m pytest tests -m gpu -q \
    -p no:cacheprovider -k "races or traces or kernels or pipeline or configs or cache or edges" \
    > gpurun_out/pytest_checks.log 2>&1
echo checks_pytest=$?
tail -5 gpurun_out/pytest_checks.log
grep -c "ARTEMIS_DCHECK failed" gpurun_out/pytest_checks.log
timeout 600 python -m pytest tests/test_gpu_races.py -q -p no:cacheprovider > gpurun_out/pytest_races.log 2>&1
echo races=$?
tail -3 gpurun_out/pytest_races.log

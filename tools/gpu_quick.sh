# Focused GPU session: selected tests (verbose, per-test timeout) + the headline bench.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout ${PYTEST_BUDGET:-1500} python -m pytest ${PYTEST_TARGETS:-tests} -m gpu -v --timeout ${PYTEST_TIMEOUT:-600} --durations=20 ${PYTEST_ARGS:-} > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err

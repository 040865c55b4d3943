# Iteration session: focused tests, the C2 bench, one ncu capture of the page kernel.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest ${PYTEST_TARGETS} -m gpu -v --timeout 600 --durations=15 > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_iter.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:${KREGEX:-k_eval_page}" -c 1 -o gpurun_out/${NAME:-page_c2} \
  python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${NAME:-page_c2}.log 2>&1

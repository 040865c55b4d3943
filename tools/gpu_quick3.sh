python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize.py -m gpu -q --timeout 600 -k "page or c1_full or c2_full or c2r or c4 or slice_codes" > gpurun_out/pytest_q3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q3.log
for c in ${CONFIGS:-c2 c2r c4}; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done

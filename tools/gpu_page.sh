# page-kernel parity iteration: the page tests, full-size C1/C2/C2r, the debug-code parity
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_fullsize.py tests/test_gpu_runtime.py -m gpu -q --timeout 900 \
  -k "page or c1_full or c2_full or c2r or slice_codes or canar" > gpurun_out/pytest_page.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_page.log
for c in ${CONFIGS:-c2}; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done

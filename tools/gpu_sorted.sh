# sorted-kernel iteration: parity tests touching the sorted kernel, then the C3 bench line
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_fullsize.py tests/test_gpu_runtime.py tests/test_sim_gpu.py -m gpu -q --timeout 900 \
  -k "sorted or rand or word or c3 or c5 or slice_codes or canar or fuzz or weak or batch" > gpurun_out/pytest_sorted.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_sorted.log
timeout 600 python bench.py --config c3 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err

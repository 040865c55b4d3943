# One GPU session: build, the GPU test suite, the headline bench + the reference arm.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2700 python -m pytest tests -m gpu -q --durations=30 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --config c2r --steps 10 --warmup 3 > gpurun_out/bench_c2r.json 2> gpurun_out/bench_c2r.err
timeout 600 python bench.py --config c1 --steps 20 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_c2.json 2> gpurun_out/ref_c2.err

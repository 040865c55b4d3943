# Final-state check: the whole GPU suite, smoke, default bench + reference arm, C1 / C4 lines.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for c in c1 c4; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_c2.json 2> gpurun_out/ref_c2.err

# Final-state check (round 2 close): GPU suite, smoke, default bench (C2 with the CPU
# baselines), C1 / C2r / C4 / C3 lines, the reference arm, the driver-style launch list.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for c in c1 c2r c4; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 python bench.py --config c3 --steps 3 --warmup 1 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_c2.json 2> gpurun_out/ref_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1

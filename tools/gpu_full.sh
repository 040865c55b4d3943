# Full session: the whole GPU suite, every config's bench line, the reference arm,
# the driver-style ncu launch list and ncu captures of the C3 / C4 / C5 kernels.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q --timeout 900 --durations=40 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in c2 c1 c2r c4; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 900 python bench.py --config c3 --steps 3 --warmup 1 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 1200 python bench.py --config c5 --steps 3 --warmup 1 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_c2.json 2> gpurun_out/ref_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k "regex:k_eval_sorted" -c 1 -o gpurun_out/sorted_c3 python bench.py --config c3 --assign 2097152 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_eval_slice_wc" -c 1 -o gpurun_out/slicewc_c4 python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c4.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k "regex:k_eval_sorted" -c 1 -o gpurun_out/sorted_c5 python bench.py --config c5 --assign 16384 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c5.log 2>&1

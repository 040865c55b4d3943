# C2 evidence after a page-kernel change: default bench line, driver-style launch list, one ncu --set full capture
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_eval_page" -c 1 -o gpurun_out/page_c2_final python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/page_c2_final.log 2>&1
echo "ncu rc=$?" >> gpurun_out/page_c2_final.log

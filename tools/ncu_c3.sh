python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 420 ncu --set full --import-source on --clock-control none -k "regex:k_eval_sorted" -c 1 -o gpurun_out/sorted_c3 python bench.py --config c3 --assign 1048576 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c3.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_c3.log

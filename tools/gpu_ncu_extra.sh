# ncu captures of the C2r page kernel (full batch) and the C3 sorted kernel (2^21-word sample)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_eval_page" -c 1 -o gpurun_out/page_c2r python bench.py --config c2r --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c2r.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_c2r.log
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_eval_sorted" -c 1 -o gpurun_out/sorted_c3_2M python bench.py --config c3 --assign 2097152 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c3.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_c3.log

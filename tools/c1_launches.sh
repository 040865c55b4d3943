python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.per_cycle_active,launch__grid_size,smsp__inst_executed.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_c1.csv python bench.py --config c1 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c1.log 2>&1

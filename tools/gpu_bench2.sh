# two back-to-back bench runs per config (noise check)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in ${CONFIGS:-c2 c2r}; do for k in 1 2; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_$k.json 2> gpurun_out/bench_${c}_$k.err; done; done

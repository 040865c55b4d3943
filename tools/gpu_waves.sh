# grid-policy sweep of the page kernel on C2 (PZX_WAVES)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for w in ${WAVES:-16 32 64 128}; do PZX_WAVES=$w timeout 300 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/waves_$w.json 2> gpurun_out/waves_$w.err; done

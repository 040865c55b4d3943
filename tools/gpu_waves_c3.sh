# grid-policy sweep of the sorted kernel on C3 (PZX_WAVES)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for w in ${WAVES:-32 64 128}; do PZX_WAVES=$w timeout 400 python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/wavesc3_$w.json 2> gpurun_out/wavesc3_$w.err; done

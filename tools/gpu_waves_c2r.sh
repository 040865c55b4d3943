python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for w in ${WAVES:-32 64 128}; do PZX_WAVES=$w timeout 300 python bench.py --config c2r --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/wavesr_$w.json 2> gpurun_out/wavesr_$w.err; done

python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for m in 512 128 32 8; do echo "min_chunk_rows=$m" >> gpurun_out/sweep_c1.log; PZX_MIN_CHUNK_ROWS=$m timeout 300 python bench.py --config c1 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'])" >> gpurun_out/sweep_c1.log; done
for m in 512 128; do echo "c4 min_chunk_rows=$m" >> gpurun_out/sweep_c1.log; PZX_MIN_CHUNK_ROWS=$m timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['kernel'])" >> gpurun_out/sweep_c1.log; done

# ncu --set full capture of one launch of a kernel (regex $KREGEX) in a short bench run of $CONFIG.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:${KREGEX:-k_eval_page}" -c 1 -o gpurun_out/${NAME:-page_c2} \
  python bench.py --config ${CONFIG:-c2} --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${NAME:-page_c2}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${NAME:-page_c2}.log

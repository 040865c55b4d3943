"""Throughput of the exact (integer-ring) path on the full C2 table, through the C ABI
(wall time of the synchronous pzx_evaluate_exact_range call, D2H included)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_06777_b200 as P
from paper_2403_06777_b200 import synth
e = synth.generate_config(synth.CONFIGS["c2"])
with P.Context(0) as ctx:
    t = ctx.compile_bit_table(e)
    for n in (1<<14, 1<<16, 1<<18):
        ctx.evaluate_exact_range(t, 0, 1024)
        t0 = time.time(); ex = ctx.evaluate_exact_range(t, 0, n); dt = time.time() - t0
        print("exact c2 n", n, "s", round(dt, 3), "evals/s %.3g" % (n / dt), "row-evals/s %.3g" % (n * t.n_rows / dt))

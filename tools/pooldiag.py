import sys, numpy as np
sys.path.insert(0, '.')
import paper_2403_06777_b200 as P
from paper_2403_06777_b200 import synth
c = P.Context(0)
e = synth.generate(20, 2000, 8, 30, 5)
t = c.compile_bit_table(e)
for n in (64, 4096, 1 << 16):
    w = np.random.default_rng(0).integers(0, 1 << 20, n, dtype=np.uint64)
    try:
        a = c.evaluate_batch(t, w)
        print(n, "ok", c.last_kernel())
    except Exception as ex:
        print(n, "FAIL", ex)
try:
    a = c.evaluate_range(t, 0, 1 << 20)
    print("range ok", c.last_kernel())
except Exception as ex:
    print("range FAIL", ex)

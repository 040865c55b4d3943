"""Per-call wall time of pzx_evaluate (pinned host buffers, C1 table) with and
without the graph replay path; run twice: PZX_NO_GRAPHS=1 and default."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_06777_b200 as P  # noqa: E402
from paper_2403_06777_b200 import _native as NV, synth  # noqa: E402

ctx = P.Context(0)
cfg = synth.CONFIGS["c1"]
t = ctx.compile_bit_table(synth.generate_config(cfg))
n = cfg.n_assign
L = NV.lib()
w = torch.arange(0, n, dtype=torch.int64).pin_memory()
amp = torch.empty(2 * n, dtype=torch.float64).pin_memory()
prob = torch.empty(n, dtype=torch.float64).pin_memory()


def call():
    st = L.pzx_evaluate(ctx.handle, t.handle, C.cast(w.data_ptr(), C.POINTER(C.c_uint64)), n,
                        C.cast(amp.data_ptr(), NV.dblp), C.cast(prob.data_ptr(), NV.dblp), P.PROB_ABS2)
    assert st == 0, L.pzx_last_error(ctx.handle).decode()


for _ in range(10):
    call()
torch.cuda.synchronize()
t0 = time.perf_counter()
K = 2000
for _ in range(K):
    call()
el = time.perf_counter() - t0
print(f"graphs={'off' if os.environ.get('PZX_NO_GRAPHS') == '1' else 'on'}: {1e6 * el / K:.1f} us per call, "
      f"{n * K / el:.3e} evals/s, kernel {ctx.last_kernel()}")

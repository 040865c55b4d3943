"""Measure the B200 pipe rates the roofline uses (SURVEY §8d asks for the
table figures to be confirmed on the box): int32 LOP3, POPC, fp64 FMA and
shared-memory loads, per SM per clock at the sampled SM clock.

    python -m paper_2403_06777_b200.microbench [out.json]
"""
from __future__ import annotations

import ctypes as C
import json
import subprocess
import sys

from . import _native as N

PIPES = {0: "lop3_int32", 1: "popc", 2: "dfma_fp64", 3: "lds32"}


def measure(device: int = 0) -> dict:
    L = N.lib()
    out = {}
    for k, name in PIPES.items():
        v = C.c_double()
        st = L.pzx_microbench(device, k, C.byref(v))
        if st:
            raise RuntimeError(f"microbench {name}: status {st}")
        out[name] = v.value
    try:
        mhz = float(subprocess.run(["nvidia-smi", "-i", str(device), "--query-gpu=clocks.max.sm",
                                    "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                   timeout=20).stdout.strip())
    except Exception:
        mhz = 1965.0
    n_sm = 148
    res = {"device": device, "sm_max_mhz": mhz, "n_sm": n_sm, "ops_per_s": out,
           "per_sm_per_clk": {k: v / (n_sm * mhz * 1e6) for k, v in out.items()},
           "how": "pzx_microbench: 8 independent dependency chains per thread x 4096 iterations, 64 warps/SM, "
                  "best of 3 timed launches (CUDA events); per-SM-per-clock at the max SM clock"}
    return res


if __name__ == "__main__":
    r = measure()
    js = json.dumps(r, indent=1)
    print(js)
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(js + "\n")

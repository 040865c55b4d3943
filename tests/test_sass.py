"""SASS invariants of the built library (CPU: cuobjdump on the sm_100a cubin,
no GPU). They pin properties the measured performance depends on and that a
small source change can silently lose: the page kernel's
G-row loops address shared memory through the uniform datapath (`LDS [UR]`;
a T table addressed from the dynamic shared base once moved them off it and
cost 8 %), its rows arrive by TMA bulk copies, and its accumulators live in
tensor memory."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2403_06777_b200", "libpzx_gpu.so")
CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"


@pytest.fixture(scope="module")
def page_sass():
    if not os.path.exists(LIB) or not os.path.exists(CUOBJDUMP):
        pytest.skip("library or cuobjdump missing")
    out = subprocess.run([CUOBJDUMP, "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs = re.split(r"\n\s*Function : ", out)
    page = [f for f in funcs if re.match(r"\S*k_eval_pageILb0E", f)]
    assert len(page) == 1
    return page[0]


def test_page_kernel_row_loops_use_the_uniform_datapath(page_sass):
    uniform = len(re.findall(r"LDS(?:\.\w+)* R\d+, \[UR", page_sass))
    assert uniform >= 24, f"only {uniform} uniform-address shared loads in k_eval_page"


def test_page_kernel_tma_and_tmem(page_sass):
    assert "UBLKCP" in page_sass          # cp.async.bulk (TMA) page loads
    assert "SYNCS" in page_sass           # mbarrier waits
    assert "LDTM" in page_sass and "STTM" in page_sass  # tcgen05.ld / st accumulators


def test_page_kernel_has_no_local_spills(page_sass):
    assert not re.search(r"\bSTL\b|\bLDL\b", page_sass)

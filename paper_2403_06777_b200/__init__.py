"""B200-native evaluator for the parametric sum-over-Cliffords scalar of arXiv 2403.06777.

Product surface (all evaluation runs in sm_100a kernels of ``libpzx_gpu.so``):

* :mod:`.pzx` -- the reference-shaped API (ParamPhase, Subterm, RingQuad,
  ScalarExpression, Context.compile_bit_table / evaluate_batch / evaluate).
* :mod:`.synth` -- seeded synthetic term tables for the BASELINE configs.
* :mod:`.dist` -- one-process-per-GPU sharding (assignment shards, term split
  with an all-reduce of partial amplitudes) over torch.distributed.
"""
from .pzx import *  # noqa: F401,F403
from .pzx import __all__ as _pzx_all

__all__ = list(_pzx_all)

"""Multi-GPU plumbing: one process per GPU over torch.distributed.

Two ways to spread the evaluation of S(a) = sum_t C_t prod_r V_tr(a):

* **assignment shards** (the default, C1-C3): every rank holds the whole table
  and evaluates a contiguous slice of the assignment batch. There is no
  collective on the data path; results are only gathered if the caller wants
  them on one rank.
* **term split** (C4/C5, a table too large for one GPU or a batch too small to
  fill it): rank r holds the terms [t_r, t_{r+1}) -- ranges balanced by ROW
  count, not term count -- evaluates partial amplitudes for the whole batch,
  and ONE all-reduce (sum) over NCCL/NVLink combines them. Probabilities are
  computed after the reduction (|sum|^2, not sum |.|^2). ``deterministic=True``
  replaces the all-reduce by an all-gather + rank-ordered sum, which is
  bit-identical for every world size that yields the same term ranges.

The per-rank compute is a ``partial_fn`` so the same collective code runs with
the CUDA evaluator (``gpu_partial_fn``) on B200s and with any CPU stand-in in
the gloo tests.
"""
from __future__ import annotations

from typing import Callable

import numpy as np
import torch
import torch.distributed as dist


def assignment_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [begin, end) slice of an n-assignment batch for `rank`."""
    return n * rank // world, n * (rank + 1) // world


def term_ranges(term_row_offset: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Split terms into `world` contiguous ranges with ~equal ROW counts."""
    off = np.asarray(term_row_offset, dtype=np.int64)
    m = len(off) - 1
    total = int(off[-1] - off[0])
    cuts = [0]
    for r in range(1, world):
        target = off[0] + total * r // world
        k = int(np.searchsorted(off, target, side="left"))
        cuts.append(min(max(k, cuts[-1]), m))
    cuts.append(m)
    return [(cuts[i], cuts[i + 1]) for i in range(world)]


def combine_partials(partial: torch.Tensor, group=None, deterministic: bool = False) -> torch.Tensor:
    """Sum per-rank partial amplitudes (float64 [2n], re/im interleaved) over ranks."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return partial
    if not deterministic:
        dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
        return partial
    parts = [torch.empty_like(partial) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, partial, group=group)
    out = parts[0].clone()
    for p in parts[1:]:
        out += p
    return out


def probabilities(amp: torch.Tensor, real: bool = False) -> torch.Tensor:
    a = amp.view(-1, 2)
    return a[:, 0].clone() if real else a[:, 0] * a[:, 0] + a[:, 1] * a[:, 1]


def evaluate_term_split(partial_fn: Callable[[int, int], torch.Tensor], term_row_offset: np.ndarray,
                        group=None, deterministic: bool = False) -> torch.Tensor:
    """Term-split evaluation: each rank computes partial_fn(t0, t1) for its row-balanced
    term range, then one all-reduce combines the partial amplitudes."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    t0, t1 = term_ranges(term_row_offset, world)[rank]
    return combine_partials(partial_fn(t0, t1), group, deterministic)


def combine_exact_partials(partial: torch.Tensor, sum_fn: Callable[[torch.Tensor], torch.Tensor],
                           group=None) -> torch.Tensor:
    """Exact term-split combine ("exact: ncclAllGather + a rank-ordered
    sum"): every rank's canonical RingQuads (int64 [n, 5]) are all-gathered
    rank-major into [world, n, 5] and summed exactly by ``sum_fn`` (on B200s
    ``gpu_exact_sum_fn``: the ``pzx_ringquad_sum_device`` kernel). An exact sum
    has one canonical value, so the result is identical for every world size."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return partial
    world = dist.get_world_size(group)
    parts = [torch.empty_like(partial) for _ in range(world)]
    dist.all_gather(parts, partial.contiguous(), group=group)
    return sum_fn(torch.stack(parts))


def evaluate_term_split_exact(partial_fn: Callable[[int, int], torch.Tensor], term_row_offset: np.ndarray,
                              sum_fn: Callable[[torch.Tensor], torch.Tensor], group=None) -> torch.Tensor:
    """Exact term split: partial_fn(t0, t1) -> canonical RingQuads [n, 5] of this
    rank's row-balanced term range, combined by combine_exact_partials."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    t0, t1 = term_ranges(term_row_offset, world)[rank]
    return combine_exact_partials(partial_fn(t0, t1), sum_fn, group)


def gather_shards(local: torch.Tensor, n_total: int, width: int = 1, group=None) -> torch.Tensor:
    """All-gather contiguous per-rank result slices (`width` values per assignment).
    Output plumbing after the evaluation, not part of the hot path."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local
    world = dist.get_world_size(group)
    sizes = [width * (e - b) for b, e in (assignment_range(n_total, world, r) for r in range(world))]
    buf = torch.zeros(max(sizes), dtype=local.dtype, device=local.device)
    buf[:local.numel()] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)])


def gpu_partial_fn(ctx, expr, n: int, first: int = 0, d_words: torch.Tensor | None = None,
                   device: int | None = None):
    """partial_fn backed by the CUDA evaluator: uploads this rank's term slice
    of `expr` and evaluates the whole batch into a device tensor."""
    def fn(t0: int, t1: int) -> torch.Tensor:
        dev = torch.device("cuda", ctx.device if device is None else device)
        out = torch.zeros(2 * n, dtype=torch.float64, device=dev)
        if t1 > t0:
            table = ctx.compile_bit_table(expr.slice_terms(t0, t1))
            ctx.evaluate_device(table, n, d_assignments=d_words.data_ptr() if d_words is not None else 0,
                                first=first, d_amp=out.data_ptr(), stream=torch.cuda.current_stream(dev).cuda_stream)
            torch.cuda.synchronize(dev)
            table.free()
        return out
    return fn


def gpu_exact_partial_fn(ctx, expr, words: np.ndarray, device: int | None = None):
    """Exact partial_fn backed by the CUDA evaluator: canonical RingQuads of this
    rank's term slice at every word, as an int64 [n, 5] device tensor."""
    def fn(t0: int, t1: int) -> torch.Tensor:
        dev = torch.device("cuda", ctx.device if device is None else device)
        if t1 <= t0:
            return torch.zeros((len(words), 5), dtype=torch.int64, device=dev)
        table = ctx.compile_bit_table(expr.slice_terms(t0, t1))
        try:
            out = ctx.evaluate_exact(table, words, allow_overflow=True)
        finally:
            table.free()
        return torch.from_numpy(out).to(dev)
    return fn


def gpu_exact_sum_fn(ctx, device: int | None = None):
    """sum_fn for combine_exact_partials: the pzx_ringquad_sum_device kernel on
    the gathered [world, n, 5] device tensor (exp = -1 marks overflow)."""
    def fn(parts: torch.Tensor) -> torch.Tensor:
        dev = torch.device("cuda", ctx.device if device is None else device)
        parts = parts.to(dev).contiguous()
        out = torch.empty(parts.shape[1:], dtype=torch.int64, device=dev)
        ctx.ringquad_sum_device(parts.data_ptr(), parts.shape[0], parts.shape[1], out.data_ptr(),
                                stream=torch.cuda.current_stream(dev).cuda_stream)
        torch.cuda.synchronize(dev)
        return out
    return fn

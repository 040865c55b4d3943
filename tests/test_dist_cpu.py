"""Multi-process (world_size 2, gloo, CPU) tests of the multi-GPU plumbing.

The per-rank compute is the CPU oracle here (the GPU kernels are covered by
the -m gpu tests); what is tested is the sharding arithmetic and the
collectives that combine per-rank results: term split + all-reduce of partial
amplitudes (and its deterministic all-gather variant), assignment shards +
gather.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_06777_b200 import dist as D
from paper_2403_06777_b200 import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.join(os.path.dirname(here), "oracle"))
    import oracle_py as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        e = synth.generate(9, 60, 4, 30, 99)
        words = np.arange(512, dtype=np.uint64)

        def partial_fn(t0, t1):
            if t1 <= t0:
                return torch.zeros(2 * len(words), dtype=torch.float64)
            _, amp = O.eval_batch(e.slice_terms(t0, t1), words, 2)
            return torch.from_numpy(amp.view(np.float64).copy())

        summed = D.evaluate_term_split(partial_fn, e.term_offset)
        det = D.evaluate_term_split(partial_fn, e.term_offset, deterministic=True)
        a0, a1 = D.assignment_range(len(words), world, rank)
        _, mine = O.eval_batch(e, words[a0:a1], 1)
        gathered = D.gather_shards(torch.from_numpy(mine.view(np.float64).copy()), len(words), width=2)
        if rank == 0:
            _, full = O.eval_batch(e, words, 2)
            q.put((summed.numpy().view(np.complex128), det.numpy().view(np.complex128),
                   gathered.numpy().view(np.complex128), full))
    finally:
        dist.destroy_process_group()


def test_term_split_and_assignment_shards_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    summed, det, gathered, full = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    scale = np.maximum(np.abs(full), np.sqrt(np.mean(np.abs(full) ** 2)))
    assert np.max(np.abs(summed - full) / scale) < 1e-12
    assert np.array_equal(summed, det)  # two ranks: both orders sum the same two numbers
    assert np.array_equal(gathered, full)


def _oracle_ring_sum(O):
    def fn(parts):
        p = parts.numpy()
        out = np.zeros(p.shape[1:], np.int64)
        for i in range(p.shape[1]):
            acc = tuple(int(v) for v in p[0, i])
            for r in range(1, p.shape[0]):
                acc = O.ring_add(acc, tuple(int(v) for v in p[r, i]))
            out[i] = acc[:5]
        return torch.from_numpy(out)
    return fn


def _exact_worker(rank, world, port, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.join(os.path.dirname(here), "oracle"))
    import oracle_py as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        e = synth.generate(9, 40, 2, 20, 7)
        words = np.arange(300, dtype=np.uint64)

        def partial_fn(t0, t1):
            if t1 <= t0:
                return torch.zeros((len(words), 5), dtype=torch.int64)
            return torch.from_numpy(O.eval_batch(e.slice_terms(t0, t1), words, 2)[0])

        got = D.evaluate_term_split_exact(partial_fn, e.term_offset, _oracle_ring_sum(O))
        if rank == 0:
            q.put((got.numpy(), O.eval_batch(e, words, 2)[0]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exact_term_split_world(world):
    """Exact term split: all-gathered canonical partials summed exactly equal the
    whole table's canonical values (bit-identical, any world size)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exact_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, full = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(got, full)


def test_term_ranges_balance_rows():
    off = np.concatenate([[0], np.cumsum(np.random.default_rng(0).integers(1, 64, 10000))])
    for world in (1, 2, 3, 8):
        rs = D.term_ranges(off, world)
        assert rs[0][0] == 0 and rs[-1][1] == 10000
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        rows = [off[t1] - off[t0] for t0, t1 in rs]
        assert max(rows) - min(rows) <= 2 * 64
    assert D.assignment_range(10, 3, 0) == (0, 3) and D.assignment_range(10, 3, 2) == (6, 10)

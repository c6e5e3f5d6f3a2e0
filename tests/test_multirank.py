"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: root ownership partitions the
roots exactly, per-rank counts summed by the one all-reduce equal the single-rank total,
and step times are reduced with MAX.  Per-rank counts come from the oracle restricted to
the rank's roots (the device path applies the same ownership rule in k_roots; its GPU
test is test_gpu_parity.py::test_rank_partition_sums_to_total)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gminputs as gi
from paper_2604_10601_b200 import partition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import OracleGraph
        n, s, d = gi.er_edges(400, 7, seed=3)
        lab = gi.uniform_labels(n, 2, 3)
        og = OracleGraph(n, s, d, lab)
        queries = [gi.tailed_triangle((0, 1, 0, 1)), gi.Query(3, [(0, 1), (1, 2)], [0, 1, 0]), gi.cycle(4)]
        counts = torch.zeros(len(queries), dtype=torch.int64)
        for i, q in enumerate(queries):
            roots = partition.owned_roots(np.flatnonzero(lab == q.labels[0]), rank, world, chunk=16)
            counts[i] = sum(og.count(q, fixed=(0, int(v))) for v in roots)
        exact = partition.reduce_counts(counts)
        t = partition.max_over_ranks(1.0 + rank)
        # uint64 counts near 2^64 (stored bit for bit in int64): the exact sum exceeds int64
        big = torch.tensor([(2**64 - 5 - (1 << 64)), 2**63 + 7 - (1 << 64), 3], dtype=torch.int64)
        big_tot = partition.reduce_counts(big)
        if rank == 0:
            totals = [og.count(q) for q in queries]
            out.put((counts.tolist(), totals, t, exact, big_tot))
    finally:
        dist.destroy_process_group()


def test_ownership_is_a_partition():
    v = np.arange(10_000)
    for world in (1, 2, 3, 8):
        own = partition.owner(v, world, chunk=64)
        assert own.min() >= 0 and own.max() < world
        parts = [partition.owned_roots(v, r, world) for r in range(world)]
        assert sum(len(p) for p in parts) == len(v)
        assert np.array_equal(np.sort(np.concatenate(parts)), v)


@pytest.mark.parametrize("world", [2])
def test_gloo_two_ranks_reduce_to_total(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    counts, totals, t, exact, big_tot = got
    assert counts == totals and exact == totals
    assert t == float(world)      # max over ranks of 1 + rank
    # uint64 inputs near 2^64 on every rank: exact sums, beyond the int64 range
    assert big_tot == [world * (2**64 - 5), world * (2**63 + 7), world * 3]

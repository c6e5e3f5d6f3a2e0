"""Host-side multi-GPU plumbing: root ownership and the per-step count reduction.

The ownership rule is the one k_roots applies on the device (include/gmatch.h,
gm_run_opts.rank/world/root_chunk): root vertex v belongs to rank (v // chunk) % world.
Every rank holds a replica of the CSR, searches the embeddings rooted at its own roots,
and the per-query counts of all ranks are summed with ONE all-reduce per step
(north_star: "per-GPU counts are reduced with one NCCL allreduce over NVLink").
"""
from __future__ import annotations

import numpy as np

DEFAULT_CHUNK = 64


def owner(v, world: int, chunk: int = DEFAULT_CHUNK):
    """Rank owning root vertex v (scalar or numpy array)."""
    return (np.asarray(v, dtype=np.int64) // chunk) % world


def owned_roots(candidates, rank: int, world: int, chunk: int = DEFAULT_CHUNK) -> np.ndarray:
    """The subset of root candidates rank `rank` searches."""
    c = np.asarray(candidates)
    return c[owner(c, world, chunk) == rank]


def reduce_count_halves(counts, group=None):
    """The step's one collective: sum per-query counts over all ranks, exactly.

    `counts` is an int64 tensor holding each rank's uint64 counts bit for bit (gm_count
    writes uint64; values >= 2^63 read as negative int64).  A plain int64 all-reduce would
    wrap once a total passes 2^63, so each count is split into 32-bit halves and both
    halves are summed in ONE all-reduce (no overflow below 2^31 ranks).  Returns the
    reduced halves (device tensor, no host sync); count_totals() reassembles them."""
    import torch
    import torch.distributed as dist
    c = counts.reshape(-1).to(torch.int64)
    halves = torch.cat([c & 0xFFFFFFFF, (c >> 32) & 0xFFFFFFFF])
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(halves, group=group)
    return halves


def count_totals(halves):
    """Exact per-query totals (Python ints, unbounded) from reduce_count_halves()."""
    h = halves.tolist()
    n = len(h) // 2
    return [h[i] + (h[n + i] << 32) for i in range(n)]


def reduce_counts(counts, group=None):
    """reduce_count_halves + count_totals; also leaves `counts` holding the totals mod 2^64
    (as int64 bit patterns)."""
    import torch
    totals = count_totals(reduce_count_halves(counts, group))
    wrapped = [t % (1 << 64) for t in totals]
    counts.copy_(torch.tensor([w - (1 << 64) if w >= 1 << 63 else w for w in wrapped],
                              dtype=counts.dtype).reshape(counts.shape))
    return totals


def as_int64_bits(values):
    """uint64 Python ints -> the int64 values with the same bits (for int64 tensors)."""
    return [v - (1 << 64) if v >= 1 << 63 else v for v in values]


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar (e.g. a device time) over all ranks."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())

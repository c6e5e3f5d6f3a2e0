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


def reduce_counts(counts, group=None):
    """Sum a per-query int64 count tensor over all ranks in place (the step's one collective)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(counts, group=group)
    return counts


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar (e.g. a device time) over all ranks."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())

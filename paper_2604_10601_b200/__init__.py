"""B200-native fine-grained subgraph matching (gMatch, arXiv 2604.10601) -- Python binding.

The binding mirrors the C ABI (include/gmatch.h) name for name:

    g = gm_load_graph(n, src, dst, labels=None, num_labels=1)     # -> Graph
    p = gm_plan_query(g, query, order=None, filter="nlf")         # -> Plan
    c, stats = gm_count(p, tau=..., rank=0, world=1, steal=True, out=None)
    rows, c, stats = gm_enumerate(p, capacity)

Host arrays are numpy; device arrays are torch CUDA tensors (PyTorch provides device
memory, streams and process groups only).  All computation happens in libgmatch.so.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib as L
from ._lib import GMError, FILTERS, GM_TIMEOUT

__all__ = ["gm_load_graph", "gm_plan_query", "gm_count", "gm_enumerate", "Graph", "Plan", "GMError",
           "version"]


def _stream_handle(stream):
    if stream is not None:
        return ctypes.c_void_p(int(stream))
    try:
        import torch
        if torch.cuda.is_available():
            return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    except ImportError:
        pass
    return ctypes.c_void_p(0)


def _is_torch_cuda(x):
    return hasattr(x, "is_cuda") and getattr(x, "is_cuda", False)


def _ptr_u32(x, n_expected=None):
    """(pointer, mem, keepalive) for a numpy array or a torch CUDA tensor of 32-bit ints."""
    if x is None:
        return ctypes.c_void_p(0), L.GM_MEM_HOST, None
    if _is_torch_cuda(x):
        import torch
        if x.dtype not in (torch.int32, torch.uint32):
            raise TypeError("device arrays must be int32/uint32 torch tensors")
        x = x.contiguous()
        if n_expected is not None and x.numel() != n_expected:
            raise ValueError("device array has the wrong length")
        return ctypes.c_void_p(x.data_ptr()), L.GM_MEM_DEVICE, x
    a = np.ascontiguousarray(x, dtype=np.uint32)
    if n_expected is not None and a.size != n_expected:
        raise ValueError("host array has the wrong length")
    return ctypes.c_void_p(a.ctypes.data), L.GM_MEM_HOST, a


def version() -> str:
    return L.lib().gm_version().decode()


class Graph:
    """Handle of a device data graph (label-partitioned CSR)."""

    def __init__(self, handle, n, num_labels):
        self._h = ctypes.c_void_p(handle)
        self.n = n
        self.num_labels = num_labels

    def info(self) -> dict:
        inf = L.GraphInfo()
        L.check(L.lib().gm_graph_info(self._h, ctypes.byref(inf)))
        return {k: getattr(inf, k) for k, _ in inf._fields_}

    def build_hubs(self, budget_bytes=64 << 20, min_degree=64, summary=-1, stream=None):
        """Rebuild the hub adjacency index (budget 0 removes it); summary level: -1 when the
        index exceeds L2, 0 never, 1 always."""
        L.check(L.lib().gm_graph_build_hubs(self._h, int(budget_bytes), int(min_degree), int(summary),
                                            _stream_handle(stream)))

    def export(self):
        """(offs, nbr, labels) copied to host numpy arrays."""
        inf = self.info()
        offs = np.zeros(inf["n"] * inf["num_labels"] + 1, np.uint32)
        nbr = np.zeros(max(inf["num_adj"], 1), np.uint32)
        lab = np.zeros(max(inf["n"], 1), np.uint32)
        L.check(L.lib().gm_graph_export(self._h, offs.ctypes.data, nbr.ctypes.data, lab.ctypes.data))
        return offs, nbr[: inf["num_adj"]], lab[: inf["n"]]

    def free(self):
        if self._h and self._h.value:
            L.lib().gm_free_graph(self._h)
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Plan:
    """Handle of a planned query (candidate bitmaps + matching order)."""

    def __init__(self, handle, graph, nq):
        self._h = ctypes.c_void_p(handle)
        self.graph = graph            # keep the graph alive while the plan lives
        self.nq = nq

    def info(self) -> dict:
        inf = L.PlanInfo()
        L.check(L.lib().gm_plan_info(self._h, ctypes.byref(inf)))
        nq = inf.nq
        return {"nq": nq, "order": list(inf.order[:nq]), "backward": list(inf.backward[:nq]),
                "cand_count": list(inf.cand_count[:nq]), "automorphisms": inf.automorphisms,
                "sb_conditions": inf.sb_conditions}

    def candidates(self, u) -> np.ndarray:
        """Boolean mask over data vertices: passed the filter for query vertex u."""
        words = np.zeros((self.graph.n + 31) // 32 or 1, np.uint32)
        L.check(L.lib().gm_plan_candidates(self._h, u, words.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))))
        bits = np.unpackbits(words.view(np.uint8), bitorder="little")
        return bits[: self.graph.n].astype(bool)

    def free(self):
        if self._h and self._h.value:
            L.lib().gm_free_plan(self._h)
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def gm_load_graph(n, src, dst, labels=None, num_labels=None, stream=None) -> Graph:
    """Build the device graph from an undirected edge list (numpy host or torch CUDA arrays)."""
    m = int(len(src))
    ps, mem_s, ks = _ptr_u32(src, m)
    pd, mem_d, kd = _ptr_u32(dst, m)
    if m and mem_s != mem_d:
        raise ValueError("src and dst must both be host or both be device arrays")
    mem = mem_s if m else L.GM_MEM_HOST
    if labels is not None:
        if num_labels is None:
            num_labels = int(labels.max()) + 1 if len(labels) else 1
        pl, mem_l, kl = _ptr_u32(labels, n)
        if mem_l != mem and m:
            raise ValueError("labels must live where src/dst live")
        mem = mem_l if not m else mem
    else:
        pl, kl = ctypes.c_void_p(0), None
        num_labels = num_labels or 1
    h = ctypes.c_void_p(0)
    L.check(L.lib().gm_load_graph(int(n), m, ps, pd, pl, int(num_labels), mem, _stream_handle(stream),
                                  ctypes.byref(h)))
    del ks, kd, kl
    return Graph(h.value, int(n), int(num_labels))


def gm_plan_query(g: Graph, query, order=None, filter="nlf", stream=None) -> Plan:
    """Plan query `query` (an object with .n, .edges (m,2), .labels) against graph g."""
    nq = int(query.n)
    qe = np.ascontiguousarray(np.asarray(query.edges, dtype=np.uint32).reshape(-1))
    ql = np.ascontiguousarray(np.asarray(query.labels, dtype=np.uint32).reshape(-1))
    u32p = ctypes.POINTER(ctypes.c_uint32)
    po = None
    if order is not None:
        oa = np.ascontiguousarray(np.asarray(order, dtype=np.uint32))
        po = oa.ctypes.data_as(u32p)
    h = ctypes.c_void_p(0)
    L.check(L.lib().gm_plan_query(g._h, nq, len(qe) // 2, qe.ctypes.data_as(u32p), ql.ctypes.data_as(u32p), po,
                                  FILTERS[filter] if isinstance(filter, str) else int(filter),
                                  _stream_handle(stream), ctypes.byref(h)))
    return Plan(h.value, g, nq)


def _opts(tau=None, rank=0, world=1, root_chunk=None, steal=True, blocks_per_sm=0, warps_per_block=0,
          time_limit_ms=0.0, roots=None, pool_bytes_max=0, set_count=True, symmetry=True, pair_count=True,
          shared_pool_ctr=None, root_seed=0, stop_at_capacity=False, team=None, no_pool=False,
          count_words=False, sibling=True, gen_cache=True):
    o = L.RunOpts()
    L.lib().gm_default_opts(ctypes.byref(o))
    if tau is not None:
        o.tau = int(tau)
    o.rank, o.world = int(rank), int(world)
    if root_chunk:
        o.root_chunk = int(root_chunk)
    o.steal = 1 if steal else 0
    o.blocks_per_sm = int(blocks_per_sm)
    if warps_per_block:
        o.warps_per_block = int(warps_per_block)
    o.time_limit_ms = float(time_limit_ms)
    keep = None
    if roots is not None:
        r = np.asarray(roots, dtype=np.uint32).reshape(-1)
        keep = np.zeros(max(1, r.size), dtype=np.uint32)   # never a NULL pointer, even when empty
        keep[: r.size] = r
        o.roots = keep.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))
        o.num_roots = r.size
    if pool_bytes_max:
        o.pool_bytes_max = int(pool_bytes_max)
    if not set_count:
        o.flags |= L.GM_FLAG_NO_SET_COUNT
    if not pair_count:
        o.flags |= L.GM_FLAG_NO_PAIR_COUNT
    if not symmetry:
        o.flags |= L.GM_FLAG_NO_SYMMETRY
    if stop_at_capacity:
        o.flags |= L.GM_FLAG_STOP_AT_CAPACITY
    if no_pool:
        o.flags |= L.GM_FLAG_NO_POOL
    if count_words:
        o.flags |= L.GM_FLAG_COUNT_WORDS
    if not sibling:
        o.flags |= L.GM_FLAG_NO_SIBLING
    if not gen_cache:
        o.flags |= L.GM_FLAG_NO_GEN_CACHE
    if team is not None:
        o.team = team._h
    if shared_pool_ctr is not None:
        o.shared_pool_ctr = ctypes.c_void_p(int(shared_pool_ctr))
    o.root_seed = int(root_seed)
    return o, keep


def gm_pool_counter_create(slots: int = 1):
    """(device pointer, IPC handle bytes) of `slots` new cross-rank pool counters on this GPU."""
    ptr = ctypes.c_void_p(0)
    h = (ctypes.c_char * L.GM_IPC_HANDLE_BYTES)()
    L.check(L.lib().gm_pool_counter_create(int(slots), ctypes.byref(ptr), h))
    return ptr.value, bytes(h)


def gm_pool_counter_open(handle: bytes):
    """Map another rank's pool counters; returns their base device pointer in this process."""
    ptr = ctypes.c_void_p(0)
    buf = (ctypes.c_char * L.GM_IPC_HANDLE_BYTES).from_buffer_copy(handle)
    L.check(L.lib().gm_pool_counter_open(buf, ctypes.byref(ptr)))
    return ptr.value


def pool_counter_slot(ptr, k: int):
    """Device pointer of counter slot k (gmatch.h: base + k * GM_POOL_COUNTER_STRIDE)."""
    return int(ptr) + int(k) * L.GM_POOL_COUNTER_STRIDE


def gm_pool_counter_reset(ptr, slots: int = 1, stream=None):
    L.check(L.lib().gm_pool_counter_reset(ctypes.c_void_p(ptr), int(slots), _stream_handle(stream)))


class Team:
    """Handle of a cross-GPU stealing team (gm_team_open); pass as gm_count(..., team=t)."""

    def __init__(self, handle, world, rank):
        self._h = ctypes.c_void_p(handle)
        self.world, self.rank = world, rank

    def free(self):
        if self._h and self._h.value:
            L.lib().gm_team_free(self._h)
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def gm_team_export() -> bytes:
    """IPC handles of this device's search workspace (control block + steal ring)."""
    h = (ctypes.c_char * L.GM_TEAM_HANDLE_BYTES)()
    L.check(L.lib().gm_team_export(h))
    return bytes(h)


def gm_team_open(world: int, rank: int, handles) -> Team:
    """Map every rank's exported workspace; handles = list of gm_team_export() bytes, rank order."""
    blob = b"".join(bytes(x) for x in handles)
    if len(blob) != world * L.GM_TEAM_HANDLE_BYTES:
        raise ValueError("need one exported handle per rank")
    buf = (ctypes.c_char * len(blob)).from_buffer_copy(blob)
    h = ctypes.c_void_p(0)
    L.check(L.lib().gm_team_open(int(world), int(rank), buf, ctypes.byref(h)))
    return Team(h.value, world, rank)


def gm_pool_counter_close(ptr, owner: bool):
    L.check(L.lib().gm_pool_counter_close(ctypes.c_void_p(ptr), 1 if owner else 0))


def gm_count(p: Plan, out=None, stream=None, **kw):
    """Count embeddings.  out: optional torch CUDA int64 tensor (1 element) receiving the
    count on the device (for an NCCL all-reduce).  Returns (count or None, stats dict)."""
    o, keep = _opts(**kw)
    st = L.RunStats()
    if out is not None:
        import torch
        if not _is_torch_cuda(out):
            raise TypeError("out must be a CUDA tensor")
        if out.dtype not in (torch.int64, torch.uint64) or out.numel() < 1 or not out.is_contiguous():
            raise TypeError("out must be a contiguous int64/uint64 CUDA tensor with at least 1 element")
        rc = L.lib().gm_count(p._h, ctypes.byref(o), ctypes.c_void_p(out.data_ptr()), L.GM_MEM_DEVICE,
                              ctypes.byref(st), _stream_handle(stream))
        L.check(rc, allow=(GM_TIMEOUT,))
        return None, st.as_dict()
    c = ctypes.c_uint64(0)
    rc = L.lib().gm_count(p._h, ctypes.byref(o), ctypes.byref(c), L.GM_MEM_HOST, ctypes.byref(st),
                          _stream_handle(stream))
    L.check(rc, allow=(GM_TIMEOUT,))
    del keep
    return int(c.value), st.as_dict()


def gm_enumerate(p: Plan, capacity: int, out=None, stream=None, **kw):
    """List up to `capacity` embeddings.  Returns (rows, total_count, stats); rows is an
    (min(capacity,total), nq) numpy array (or `out`, a torch CUDA int32 tensor, if given)."""
    o, keep = _opts(**kw)
    st = L.RunStats()
    c = ctypes.c_uint64(0)
    if out is not None:
        import torch
        if not _is_torch_cuda(out):
            raise TypeError("out must be a CUDA tensor")
        if (out.dtype not in (torch.int32, torch.uint32) or not out.is_contiguous()
                or out.numel() < int(capacity) * p.nq):
            raise TypeError("out must be a contiguous int32/uint32 CUDA tensor of at least capacity * nq elements")
        rc = L.lib().gm_enumerate(p._h, ctypes.byref(o), ctypes.c_void_p(out.data_ptr()), int(capacity),
                                  L.GM_MEM_DEVICE, ctypes.byref(c), ctypes.byref(st), _stream_handle(stream))
        L.check(rc, allow=(GM_TIMEOUT,))
        return out, int(c.value), st.as_dict()
    buf = np.zeros((max(int(capacity), 1), p.nq), np.uint32)
    rc = L.lib().gm_enumerate(p._h, ctypes.byref(o), ctypes.c_void_p(buf.ctypes.data), int(capacity),
                              L.GM_MEM_HOST, ctypes.byref(c), ctypes.byref(st), _stream_handle(stream))
    L.check(rc, allow=(GM_TIMEOUT,))
    del keep
    total = int(c.value)
    return buf[: min(int(capacity), total)], total, st.as_dict()

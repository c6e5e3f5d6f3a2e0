"""ctypes wrapper of the plain-C oracle (oracle/gm_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, never by the product package
paper_2604_10601_b200 (which must fail loudly without its CUDA library instead
of falling back here).  See gm_oracle.c's header for the definitions followed.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_u32p = ctypes.POINTER(ctypes.c_uint32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u8p = ctypes.POINTER(ctypes.c_uint8)


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, no fast-math, no OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        lib.or_graph_new.restype = ctypes.c_void_p
        lib.or_graph_new.argtypes = [ctypes.c_int64, ctypes.c_int64, _u32p, _u32p, _u32p]
        lib.or_graph_free.argtypes = [ctypes.c_void_p]
        lib.or_graph_num_adj.restype = ctypes.c_int64
        lib.or_graph_num_adj.argtypes = [ctypes.c_void_p]
        lib.or_graph_export.argtypes = [ctypes.c_void_p, _i64p, _u32p]
        lib.or_count.restype = ctypes.c_uint64
        lib.or_count.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _u32p, _u32p,
                                 ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64, _u32p, ctypes.c_uint64]
        lib.or_count_budget.restype = ctypes.c_uint64
        lib.or_count_budget.argtypes = lib.or_count.argtypes + [ctypes.c_uint64]
        lib.or_last_found.restype = ctypes.c_uint64
        lib.or_last_found.argtypes = []
        lib.or_filter.restype = ctypes.c_int
        lib.or_filter.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _u32p, _u32p,
                                  ctypes.c_int, ctypes.c_uint32, _u8p]
        _lib = lib
    return _lib


def _p(a, t=_u32p):
    return a.ctypes.data_as(t)


class OracleGraph:
    """The simple undirected labelled graph on the given (src, dst) pairs."""

    def __init__(self, n, src, dst, labels=None):
        lib = _load()
        self.n = int(n)
        self._src = np.ascontiguousarray(src, dtype=np.uint32)
        self._dst = np.ascontiguousarray(dst, dtype=np.uint32)
        self.labels = (np.zeros(self.n, dtype=np.uint32) if labels is None
                       else np.ascontiguousarray(labels, dtype=np.uint32))
        self._h = lib.or_graph_new(self.n, len(self._src), _p(self._src), _p(self._dst), _p(self.labels))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.or_graph_free(self._h)
            self._h = None

    def csr(self):
        lib = _load()
        m2 = lib.or_graph_num_adj(self._h)
        off = np.zeros(self.n + 1, dtype=np.int64)
        adj = np.zeros(max(m2, 1), dtype=np.uint32)
        lib.or_graph_export(self._h, _p(off, _i64p), _p(adj))
        return off, adj[:m2]

    def count(self, q, fixed=None, limit=0, max_nodes=0):
        """Number of embeddings of q (Definition 1); fixed=(u, v) pins M[u] = v.
        With max_nodes > 0 returns None when the search needs more tree nodes than that."""
        lib = _load()
        qe = np.ascontiguousarray(q.edges, dtype=np.uint32).reshape(-1)
        ql = np.ascontiguousarray(q.labels, dtype=np.uint32)
        fu, fv = (-1, 0) if fixed is None else (int(fixed[0]), int(fixed[1]))
        r = lib.or_count_budget(self._h, q.n, len(q.edges), _p(qe), _p(ql), fu, fv, limit, None, 0,
                                int(max_nodes))
        if r == 2 ** 64 - 1:
            raise ValueError("oracle: bad query")
        if r == 2 ** 64 - 2:
            return None
        return int(r)

    def count_budgeted(self, q, fixed=None, max_nodes=1_000_000):
        """(embeddings found, complete) after at most max_nodes search-tree nodes.  For timing
        the oracle on bounded work (bench.py cpu_baseline); not an expected value."""
        r = self.count(q, fixed=fixed, max_nodes=max_nodes)
        return int(_load().or_last_found()), r is not None

    def enumerate(self, q, fixed=None, cap=None) -> np.ndarray:
        """All embeddings as an (count, nq) array, rows sorted lexicographically."""
        total = self.count(q, fixed)
        cap = total if cap is None else min(cap, total)
        lib = _load()
        qe = np.ascontiguousarray(q.edges, dtype=np.uint32).reshape(-1)
        ql = np.ascontiguousarray(q.labels, dtype=np.uint32)
        out = np.zeros((max(cap, 1), q.n), dtype=np.uint32)
        fu, fv = (-1, 0) if fixed is None else (int(fixed[0]), int(fixed[1]))
        lib.or_count(self._h, q.n, len(q.edges), _p(qe), _p(ql), fu, fv, 0, _p(out), cap)
        out = out[:cap]
        if cap:
            out = out[np.lexsort(out.T[::-1])]
        return out

    def filter(self, q, kind: str = "nlf", num_labels=None) -> np.ndarray:
        """(nq, n) uint8 matrix: 1 iff v passes LDF (kind='ldf') or LDF+NLF (kind='nlf') for u."""
        lib = _load()
        L = int(num_labels if num_labels is not None else max(int(self.labels.max(initial=0)),
                                                                int(q.labels.max(initial=0))) + 1)
        qe = np.ascontiguousarray(q.edges, dtype=np.uint32).reshape(-1)
        ql = np.ascontiguousarray(q.labels, dtype=np.uint32)
        out = np.zeros((q.n, self.n), dtype=np.uint8)
        rc = lib.or_filter(self._h, q.n, len(q.edges), _p(qe), _p(ql), 1 if kind == "ldf" else 2, L,
                           _p(out, _u8p))
        if rc != 0:
            raise ValueError("oracle: bad query")
        return out

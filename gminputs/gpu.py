"""GPU versions of the gminputs generators (bit-identical to the numpy ones) + query growth
on device-resident edge lists.  Input generation only -- no matching arithmetic."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import (RMAT_ABC, RMAT_SCRAMBLE_ADD, RMAT_SCRAMBLE_MUL, M64, Query, rng_u64, STREAM_QUERY)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen_gpu.cu")
_LIB = os.path.join(_HERE, "libgmgen.so")
_lib = None


def build(force=False):
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-o", _LIB, _SRC])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        u64, vp, d = ctypes.c_uint64, ctypes.c_void_p, ctypes.c_double
        L.gen_rmat.argtypes = [ctypes.c_int, u64, u64, d, d, d, u64, u64, vp, vp, vp]
        L.gen_er.argtypes = [u64, u64, u64, vp, vp, vp]
        L.gen_labels.argtypes = [u64, ctypes.c_uint32, u64, vp, vp]
        L.gen_incident.argtypes = [u64, vp, vp, vp, vp, vp, vp, u64, vp]
        L.gen_neighbors.argtypes = [u64, vp, vp, ctypes.c_uint32, vp, vp, u64, vp]
        _lib = L
    return _lib


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def rmat_edges(scale, edge_factor, seed, device="cuda"):
    import torch
    n = 1 << scale
    m = edge_factor * n
    src = torch.empty(m, dtype=torch.int32, device=device)
    dst = torch.empty(m, dtype=torch.int32, device=device)
    a, b, c = RMAT_ABC
    rc = _load().gen_rmat(scale, m, seed, a, a + b, a + b + c, RMAT_SCRAMBLE_MUL & M64, RMAT_SCRAMBLE_ADD & M64,
                          src.data_ptr(), dst.data_ptr(), _stream())
    assert rc == 0, rc
    return n, src, dst


def er_edges(n, avg_deg, seed, device="cuda"):
    import torch
    m = int(round(n * avg_deg / 2))
    src = torch.empty(m, dtype=torch.int32, device=device)
    dst = torch.empty(m, dtype=torch.int32, device=device)
    assert _load().gen_er(n, m, seed, src.data_ptr(), dst.data_ptr(), _stream()) == 0
    return n, src, dst


def uniform_labels(n, num_labels, seed, device="cuda"):
    import torch
    lab = torch.empty(n, dtype=torch.int32, device=device)
    assert _load().gen_labels(n, num_labels, seed, lab.data_ptr(), _stream()) == 0
    return lab


class DeviceNeighbors:
    """neighbors(v) of the simple graph on a device-resident edge list: one scan of all
    edges per new vertex (cached), so query growth on scale-24/26 graphs needs no host CSR.
    Gives the same sorted, deduplicated lists as gminputs.HostAdjacency."""

    def __init__(self, n, src, dst):
        import torch
        self.n, self.src, self.dst = n, src, dst
        self.bits = torch.zeros((n + 31) // 32, dtype=torch.int32, device=src.device)
        self.cnt = torch.zeros(1, dtype=torch.int64, device=src.device)
        self.cache = {}

    def neighbors(self, v):
        v = int(v)
        if v in self.cache:
            return self.cache[v]
        import torch
        cap = 1 << 16
        while True:
            self.cnt.zero_()
            out = torch.empty(cap, dtype=torch.int32, device=self.src.device)
            assert _load().gen_neighbors(self.src.numel(), self.src.data_ptr(), self.dst.data_ptr(), v,
                                         out.data_ptr(), self.cnt.data_ptr(), cap, _stream()) == 0
            k = int(self.cnt.item())
            if k <= cap:
                break
            cap = 1 << int(np.ceil(np.log2(k)))
        nb = out[:k].cpu().numpy().view(np.uint32)
        nb = np.unique(nb[nb != v])
        self.cache[v] = nb
        return nb

    def induced_edges(self, vs):
        """Edges of the simple graph with both endpoints in vs, as a sorted (k, 2) array of
        (a, b) pairs with a < b (one edge scan)."""
        import torch
        self.bits.zero_()
        bits = np.zeros(self.bits.numel(), np.uint32)
        for v in vs:
            bits[v >> 5] |= np.uint32(1 << (v & 31))
        self.bits.copy_(torch.from_numpy(bits.view(np.int32)))
        cap = 1 << 22
        while True:
            self.cnt.zero_()
            os_ = torch.empty(cap, dtype=torch.int32, device=self.src.device)
            od = torch.empty(cap, dtype=torch.int32, device=self.src.device)
            assert _load().gen_incident(self.src.numel(), self.src.data_ptr(), self.dst.data_ptr(),
                                        self.bits.data_ptr(), os_.data_ptr(), od.data_ptr(), self.cnt.data_ptr(),
                                        cap, _stream()) == 0
            k = int(self.cnt.item())
            if k <= cap:
                break
            cap = 1 << int(np.ceil(np.log2(k)))
        s = os_[:k].cpu().numpy().view(np.uint32)
        d = od[:k].cpu().numpy().view(np.uint32)
        keep = np.isin(s, np.asarray(vs, np.uint32)) & np.isin(d, np.asarray(vs, np.uint32)) & (s != d)
        a, b = np.minimum(s[keep], d[keep]), np.maximum(s[keep], d[keep])
        return np.unique(np.stack([a, b], 1), axis=0) if len(a) else np.zeros((0, 2), np.uint32)

    def of_set(self, vs):
        """{v: sorted neighbour array} for every v in vs (one edge scan)."""
        import torch
        self.bits.zero_()
        bits = np.zeros(self.bits.numel(), np.uint32)
        for v in vs:
            bits[v >> 5] |= np.uint32(1 << (v & 31))
        self.bits.copy_(torch.from_numpy(bits.view(np.int32)))
        cap = 1 << 22
        while True:
            self.cnt.zero_()
            os_ = torch.empty(cap, dtype=torch.int32, device=self.src.device)
            od = torch.empty(cap, dtype=torch.int32, device=self.src.device)
            assert _load().gen_incident(self.src.numel(), self.src.data_ptr(), self.dst.data_ptr(),
                                        self.bits.data_ptr(), os_.data_ptr(), od.data_ptr(), self.cnt.data_ptr(),
                                        cap, _stream()) == 0
            k = int(self.cnt.item())
            if k <= cap:
                break
            cap = 1 << int(np.ceil(np.log2(k)))
        s = os_[:k].cpu().numpy().view(np.uint32)
        d = od[:k].cpu().numpy().view(np.uint32)
        out = {}
        vs = set(vs)
        for v in vs:
            nb = np.concatenate([d[s == v], s[d == v]])
            nb = np.unique(nb[nb != v])
            out[v] = nb
        return out

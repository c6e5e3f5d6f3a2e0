"""ctypes binding of libgmatch.so -- argument marshalling only.

Every step of the matching path runs in the CUDA library (include/gmatch.h); this
module converts numpy arrays / torch CUDA tensors into pointers, fills the C structs
and raises on error codes.  There is no Python or CPU fallback: if the library is
missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GM_LIB") or os.path.join(_HERE, "libgmatch.so")   # GM_LIB: A/B builds

GM_OK, GM_ERR_ARG, GM_ERR_CUDA, GM_ERR_NOMEM, GM_ERR_LIMIT, GM_TIMEOUT = 0, 1, 2, 3, 4, 5
GM_MEM_HOST, GM_MEM_DEVICE = 0, 1
GM_MAX_QUERY = 32
GM_FLAG_NO_SET_COUNT = 1
GM_FLAG_NO_SYMMETRY = 2
GM_FLAG_NO_PAIR_COUNT = 4
GM_FLAG_STOP_AT_CAPACITY = 8
GM_FLAG_NO_POOL = 16
GM_FLAG_COUNT_WORDS = 32
GM_FLAG_NO_SIBLING = 64
GM_FLAG_NO_GEN_CACHE = 128
GM_TEAM_HANDLE_BYTES = 256
GM_PATH_SET_COUNT, GM_PATH_PAIR_COUNT, GM_PATH_PAR_CHECKS, GM_PATH_SYMMETRY, GM_PATH_SIBLING = 1, 2, 4, 8, 16
GM_PATH_GEN_CACHE = 32
FILTERS = {"none": 0, "ldf": 1, "nlf": 2}

# every symbol include/gmatch.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "gm_load_graph", "gm_graph_info", "gm_graph_build_hubs", "gm_graph_export", "gm_free_graph",
    "gm_plan_query", "gm_plan_info", "gm_plan_candidates", "gm_free_plan",
    "gm_default_opts", "gm_count", "gm_enumerate", "gm_last_error", "gm_version",
    "gm_pool_counter_create", "gm_pool_counter_open", "gm_pool_counter_reset", "gm_pool_counter_close",
    "gm_team_export", "gm_team_open", "gm_team_free",
]
GM_IPC_HANDLE_BYTES = 64
GM_POOL_COUNTER_STRIDE = 128


class GraphInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint64), ("num_adj", ctypes.c_uint64), ("num_labels", ctypes.c_uint32),
                ("d_max", ctypes.c_uint32), ("device_bytes", ctypes.c_uint64), ("hubs", ctypes.c_uint32),
                ("hub_min_degree", ctypes.c_uint32), ("hub_bytes", ctypes.c_uint64),
                ("hub_summary_words", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("nq", ctypes.c_uint32), ("order", ctypes.c_uint32 * GM_MAX_QUERY),
                ("backward", ctypes.c_uint32 * GM_MAX_QUERY), ("cand_count", ctypes.c_uint64 * GM_MAX_QUERY),
                ("automorphisms", ctypes.c_uint64), ("sb_conditions", ctypes.c_uint32)]


class RunOpts(ctypes.Structure):
    _fields_ = [("tau", ctypes.c_uint64), ("rank", ctypes.c_uint32), ("world", ctypes.c_uint32),
                ("root_chunk", ctypes.c_uint32), ("steal", ctypes.c_uint32),
                ("blocks_per_sm", ctypes.c_uint32), ("warps_per_block", ctypes.c_uint32),
                ("time_limit_ms", ctypes.c_double), ("roots", ctypes.POINTER(ctypes.c_uint32)),
                ("num_roots", ctypes.c_uint64), ("pool_bytes_max", ctypes.c_uint64),
                ("flags", ctypes.c_uint32), ("shared_pool_ctr", ctypes.c_void_p), ("root_seed", ctypes.c_uint64),
                ("team", ctypes.c_void_p)]


class RunStats(ctypes.Structure):
    _fields_ = [("count", ctypes.c_uint64), ("roots", ctypes.c_uint64), ("pool_size", ctypes.c_uint64),
                ("pool_depth", ctypes.c_uint32), ("timed_out", ctypes.c_uint32),
                ("donations", ctypes.c_uint64), ("tasks", ctypes.c_uint64), ("rounds", ctypes.c_uint64),
                ("dfs_ms", ctypes.c_float), ("total_ms", ctypes.c_float), ("dfs_launches", ctypes.c_uint32),
                ("kernel_launches", ctypes.c_uint32), ("grid", ctypes.c_uint32), ("block", ctypes.c_uint32),
                ("words", ctypes.c_uint64), ("automorphisms", ctypes.c_uint64), ("paths", ctypes.c_uint32),
                ("stack_levels", ctypes.c_uint32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib():
    """Load libgmatch.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: build it with `python -m paper_2604_10601_b200.build` "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, u32p, u64p = ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint64)
        L.gm_load_graph.argtypes = [ctypes.c_uint64, ctypes.c_uint64, vp, vp, vp, ctypes.c_uint32, ctypes.c_int, vp,
                                    ctypes.POINTER(vp)]
        L.gm_graph_info.argtypes = [vp, ctypes.POINTER(GraphInfo)]
        L.gm_graph_export.argtypes = [vp, vp, vp, vp]
        L.gm_graph_build_hubs.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, vp]
        L.gm_free_graph.argtypes = [vp]
        L.gm_free_graph.restype = None
        L.gm_plan_query.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint32, u32p, u32p, u32p, ctypes.c_uint32, vp,
                                    ctypes.POINTER(vp)]
        L.gm_plan_info.argtypes = [vp, ctypes.POINTER(PlanInfo)]
        L.gm_plan_candidates.argtypes = [vp, ctypes.c_uint32, u32p]
        L.gm_free_plan.argtypes = [vp]
        L.gm_free_plan.restype = None
        L.gm_default_opts.argtypes = [ctypes.POINTER(RunOpts)]
        L.gm_default_opts.restype = None
        L.gm_count.argtypes = [vp, ctypes.POINTER(RunOpts), vp, ctypes.c_int, ctypes.POINTER(RunStats), vp]
        L.gm_enumerate.argtypes = [vp, ctypes.POINTER(RunOpts), vp, ctypes.c_uint64, ctypes.c_int, u64p,
                                   ctypes.POINTER(RunStats), vp]
        L.gm_pool_counter_create.argtypes = [ctypes.c_uint32, ctypes.POINTER(vp), vp]
        L.gm_pool_counter_open.argtypes = [vp, ctypes.POINTER(vp)]
        L.gm_pool_counter_reset.argtypes = [vp, ctypes.c_uint32, vp]
        L.gm_pool_counter_close.argtypes = [vp, ctypes.c_int]
        L.gm_team_export.argtypes = [vp]
        L.gm_team_open.argtypes = [ctypes.c_uint32, ctypes.c_uint32, vp, ctypes.POINTER(vp)]
        L.gm_team_free.argtypes = [vp]
        L.gm_team_free.restype = None
        L.gm_last_error.restype = ctypes.c_char_p
        L.gm_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


class GMError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"gmatch error {code}: {msg}")
        self.code = code


def check(rc, allow=()):
    if rc != GM_OK and rc not in allow:
        raise GMError(rc, lib().gm_last_error().decode())
    return rc

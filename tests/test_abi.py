"""Host-side checks of the C ABI: the library builds, loads, and exports every symbol
include/gmatch.h declares; struct layouts in the binding match the header.  No GPU needed."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "gmatch.h")).read()
    return sorted(set(re.findall(r"GM_API\s+(?:int|void|const char \*)\s*(gm_\w+)\(", txt)))


def test_library_builds_and_exports_all_declared_symbols():
    from paper_2604_10601_b200 import build as b
    lib_path = b.build()
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib_path], text=True)
    exported = set(re.findall(r" T (gm_\w+)", out))
    declared = _header_symbols()
    assert declared, "no GM_API declarations parsed"
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    from paper_2604_10601_b200 import _lib
    assert sorted(_lib.EXPORTS) == declared
    L = _lib.lib()
    for s in declared:
        assert hasattr(L, s)
    assert b"sm_100a" in L.gm_version()


def test_sm100a_cubin_present():
    from paper_2604_10601_b200 import build as b
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", b.build()], text=True)
    assert "sm_100a" in out


def test_default_opts_layout():
    from paper_2604_10601_b200 import _lib
    o = _lib.RunOpts()
    _lib.lib().gm_default_opts(ctypes.byref(o))
    assert o.tau == 1000000 and o.world == 1 and o.root_chunk == 64 and o.steal == 1
    assert o.warps_per_block == 0 and o.pool_bytes_max == 1 << 30   # 0: per query, the most resident warps
    # struct sizes match the C layout (checked with a tiny C program compiled by gcc)
    src = r'''
    #include <stdio.h>
    #include <stddef.h>
    #include "gmatch.h"
    int main(){printf("%zu %zu %zu %zu\n", sizeof(gm_run_opts), sizeof(gm_run_stats),
        sizeof(gm_plan_info_t), sizeof(gm_graph_info_t)); return 0;}
    '''
    tmp = "/tmp/gm_sizes"
    with open(tmp + ".c", "w") as f:
        f.write(src)
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", tmp, tmp + ".c"])
    sizes = [int(x) for x in subprocess.check_output([tmp], text=True).split()]
    assert sizes == [ctypes.sizeof(_lib.RunOpts), ctypes.sizeof(_lib.RunStats), ctypes.sizeof(_lib.PlanInfo),
                     ctypes.sizeof(_lib.GraphInfo)]


def test_errors_without_device_are_reported_not_fatal():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    import numpy as np
    import paper_2604_10601_b200 as gm
    with pytest.raises(gm.GMError):
        gm.gm_load_graph(3, np.array([0, 1], np.uint32), np.array([1, 2], np.uint32))

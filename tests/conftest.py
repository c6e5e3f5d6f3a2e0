import os
import re
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _expand(tok):
    """'1..50' -> [1..50]; '7' -> [7]."""
    if ".." in tok:
        a, b = tok.split("..")
        return list(range(int(a), int(b) + 1))
    return [int(tok)]


def load_fig1():
    """Parse tests/golden/fig1_example.txt -> (n, src, dst, labels, Query, expectations)."""
    from gminputs import Query
    path = os.path.join(ROOT, "tests", "golden", "fig1_example.txt")
    qn, qlab, qedges, n = 0, [], [], 0
    labels, src, dst, exp = {}, [], [], {"feasible": []}
    for raw in open(path):
        line = raw.split("#")[0].strip()
        if not line:
            continue
        key, *rest = line.split()
        if key == "query_vertices":
            qn = int(rest[0])
        elif key == "query_labels":
            qlab = [int(x) for x in rest]
        elif key == "query_edges":
            vals = [int(x) for x in rest]
            qedges = list(zip(vals[0::2], vals[1::2]))
        elif key == "data_vertices":
            n = int(rest[0])
        elif key == "label":
            for tok in rest[1:]:
                for v in _expand(tok):
                    labels[v] = int(rest[0])
        elif key == "edges":
            for tok in rest:
                a, b = tok.split("-", 1)
                bs = _expand(b.strip("{}"))
                for x in bs:
                    src.append(int(a)); dst.append(x)
        elif key == "expect_count":
            exp["count"] = int(rest[0])
        elif key == "expect_match":
            exp["match"] = [int(x) for x in rest]
        elif key == "expect_feasible_u3_given":
            i = rest.index(":")
            exp["feasible"].append(([int(x) for x in rest[:i]], [v for t in rest[i + 1:] for v in _expand(t)]))
        elif key == "expect_degree":
            exp["degree"] = (int(rest[0]), int(rest[1]))
        elif key == "expect_degree_less":
            exp["degree_less"] = (int(rest[0]), int(rest[1]))
    lab = np.array([labels[v] for v in range(n)], dtype=np.uint32)
    q = Query(qn, qedges, qlab, "fig1_tailed_triangle")
    return n, np.array(src, np.uint32), np.array(dst, np.uint32), lab, q, exp

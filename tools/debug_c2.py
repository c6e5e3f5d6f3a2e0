import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gminputs as gi
import paper_2604_10601_b200 as gm
from oracle import OracleGraph
t0 = time.time()
n, s, d = gi.rmat_edges(18, 16, 2)
lab = gi.uniform_labels(n, 8, 2)
off, nb = gi.simple_adjacency(n, s, d)
g = gm.gm_load_graph(n, s, d, lab, 8)
og = OracleGraph(n, s, d, lab)
print("setup", round(time.time() - t0, 1), g.info(), flush=True)
rs = np.random.default_rng(1)
for qs in range(4):
    q = (gi.random_query if qs % 2 == 0 else gi.random_walk_query)(off, nb, lab, 8, seed=100 + qs)
    p = gm.gm_plan_query(g, q)
    inf = p.info()
    u0 = inf["order"][0]
    cands = np.flatnonzero(p.candidates(u0))
    roots, ref = [], 0
    t = time.time()
    for v in rs.permutation(cands)[:40]:
        c = og.count(q, fixed=(u0, int(v)), max_nodes=300000)
        if c is not None:
            roots.append(int(v)); ref += c
        if len(roots) == 8:
            break
    print(qs, q.edges.tolist(), q.labels.tolist(), inf["order"], "oracle", round(time.time() - t, 1), len(roots), ref, flush=True)
    for steal in (False, True):
        for tau in (1, 1000000):
            t = time.time()
            c, st = gm.gm_count(p, roots=np.array(roots, np.uint32), tau=tau, steal=steal, time_limit_ms=20000)
            print("   steal", steal, "tau", tau, c, ref, c == ref, round(time.time() - t, 2), {k: st[k] for k in ("timed_out", "pool_size", "pool_depth", "donations", "tasks", "dfs_ms")}, flush=True)

import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gminputs as gi
import paper_2604_10601_b200 as gm
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 18
steal = int(sys.argv[2]) if len(sys.argv) > 2 else 1
n, s, d = gi.rmat_edges(scale, 16, 2)
lab = gi.uniform_labels(n, 8, 2)
off, nb = gi.simple_adjacency(n, s, d)
g = gm.gm_load_graph(n, s, d, lab, 8)
print(g.info(), flush=True)
rs = np.random.default_rng(1)
for qs in range(3):
    q = gi.random_query(off, nb, lab, 8, seed=100 + qs)
    p = gm.gm_plan_query(g, q)
    inf = p.info()
    print(q.edges.tolist(), q.labels.tolist(), inf, flush=True)
    u0 = inf["order"][0]
    cands = np.flatnonzero(p.candidates(u0))
    roots = rs.choice(cands, min(10, len(cands)), replace=False).astype(np.uint32)
    for tau in (1, 1000):
        c, st = gm.gm_count(p, roots=roots, tau=tau, steal=bool(steal))
        print(tau, c, st, flush=True)

import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gminputs as gi
import paper_2604_10601_b200 as gm
from oracle import OracleGraph
scale = int(sys.argv[1]); qk = int(sys.argv[2]); nroots = int(sys.argv[3])
n, s, d = gi.rmat_edges(scale, 8, 3)
g = gm.gm_load_graph(n, s, d)
og = OracleGraph(n, s, d)
rs = np.random.default_rng(0)
for q in [gi.path(qk), gi.cycle(qk), gi.star(qk - 1), gi.clique(min(qk, 5))]:
    p = gm.gm_plan_query(g, q)
    u0 = p.info()["order"][0]
    roots = rs.choice(n, nroots, replace=False).astype(np.uint32)
    t = time.time()
    ref = sum(og.count(q, fixed=(u0, int(v))) for v in roots)
    to = time.time() - t
    for steal in (0, 1):
        for tau in (1, 1000):
            c, st = gm.gm_count(p, roots=roots, tau=tau, steal=bool(steal))
            print(q.name, steal, tau, c, ref, "OK" if c == ref else "MISMATCH", f"oracle {to:.2f}s dfs {st['dfs_ms']:.2f}ms don {st['donations']} pool {st['pool_size']}@{st['pool_depth']}", flush=True)

import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gminputs as gi
import paper_2604_10601_b200 as gm
import bench
cfg = bench.CONFIGS["rmat18"]
n, s, d, lab = bench.make_graph_host(cfg)
off, nb = gi.simple_adjacency(n, s, d)
g = gm.gm_load_graph(n, s, d, lab, 8)
tl = float(sys.argv[1])
for kind in ("uniform_dense", "uniform", "walk"):
    for seed in range(3000, 3012):
        if kind == "uniform_dense":
            q = gi.random_query(off, nb, lab, 8, seed=seed, min_avg_degree=3.0, max_restarts=20000)
        elif kind == "uniform":
            q = gi.random_query(off, nb, lab, 8, seed=seed)
        else:
            q = gi.random_walk_query(off, nb, lab, 8, seed=seed)
        p = gm.gm_plan_query(g, q)
        c, st = gm.gm_count(p, time_limit_ms=tl)
        print(json.dumps({"kind": kind, "seed": seed, "m": len(q.edges), "count": c, "ms": round(st["total_ms"], 2),
                          "to": st["timed_out"], "tasks": st["tasks"]}), flush=True)

"""Run candidate query sets on a config and print count / time, to pick bench query seeds."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gminputs as gi
import paper_2604_10601_b200 as gm

scale, ef, nl, size, nseeds, tl = (int(x) for x in sys.argv[1:7])
t0 = time.time()
n, s, d = gi.rmat_edges(scale, ef, 2)
lab = gi.uniform_labels(n, nl, 2)
off, nb = gi.simple_adjacency(n, s, d)
print(f"gen {time.time()-t0:.1f}s", flush=True)
g = gm.gm_load_graph(n, s, d, lab, nl)
print(g.info(), flush=True)
for kind in ("dense", "sparse"):
    for seed in range(nseeds):
        try:
            q = (gi.random_query if kind == "dense" else gi.random_walk_query)(off, nb, lab, size, seed=1000 + seed)
        except RuntimeError as e:
            print(kind, seed, "gen-fail"); continue
        p = gm.gm_plan_query(g, q)
        t = time.time()
        c, st = gm.gm_count(p, time_limit_ms=tl)
        dt = time.time() - t
        print(json.dumps({"kind": kind, "seed": 1000 + seed, "m": len(q.edges), "count": c, "wall_ms": round(dt * 1e3, 2),
                          "dfs_ms": round(st["dfs_ms"], 3), "total_ms": round(st["total_ms"], 3), "to": st["timed_out"],
                          "tasks": st["tasks"], "pool": st["pool_size"], "depth": st["pool_depth"], "don": st["donations"],
                          "roots": st["roots"]}), flush=True)

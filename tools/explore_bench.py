"""Per-query completion times of a bench config's own query set under a long limit.
    python tools/explore_bench.py CONFIG LIMIT_MS [ROOT_SEED]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import gminputs as gi  # noqa: E402
import paper_2604_10601_b200 as gm  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1]]
limit = float(sys.argv[2])
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 0
n, s, d, lab = bench.make_graph_device(cfg)
lh = lab.cpu().numpy().view(np.uint32)
if cfg["kind"] != "rmat" or cfg["scale"] <= 20:
    adj = gi.HostAdjacency(*gi.simple_adjacency(n, s.cpu().numpy().view(np.uint32), d.cpu().numpy().view(np.uint32)))
else:
    import gminputs.gpu as gg
    adj = gg.DeviceNeighbors(n, s, d)
qs = bench.build_queries(cfg, adj, lh)
g = gm.gm_load_graph(n, s, d, lab, cfg["labels"])
for q in qs:
    p = gm.gm_plan_query(g, q)
    c, st = gm.gm_count(p, time_limit_ms=limit, root_seed=seed)
    print(json.dumps({"q": q.name, "m": len(q.edges), "count": c, "ms": round(st["total_ms"], 1),
                      "timed_out": st["timed_out"], "tasks": st["tasks"], "aut": st["automorphisms"],
                      "paths": st["paths"], "donations": st["donations"]}), flush=True)

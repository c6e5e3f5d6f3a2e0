"""Print the plan and one full-query run of every query of a bench config.
   python tools/plans.py [CONFIG] [LIMIT_MS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import gminputs.gpu as gg  # noqa: E402
import paper_2604_10601_b200 as gm  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "rmat18"
limit = float(sys.argv[2]) if len(sys.argv) > 2 else 1000.0
cfg = bench.CONFIGS[cfgname]
n, s, d, lab = bench.make_graph_device(cfg)
lh = lab.cpu().numpy().view(np.uint32)
adj = gg.DeviceNeighbors(n, s, d) if (cfg.get("dense") or cfg.get("sparse")) else None
qs = bench.build_queries(cfg, adj, lh)
g = gm.gm_load_graph(n, s, d, lab, cfg["labels"])
for q in qs:
    p = gm.gm_plan_query(g, q)
    inf = p.info()
    order = inf["order"]
    pos = {u: i for i, u in enumerate(order)}
    bw = []
    for i, u in enumerate(order):
        bw.append(sorted(pos[w] for a, b in q.edges for w in ((b,) if a == u else (a,) if b == u else ()) if pos[w] < i))
    c, st = gm.gm_count(p, time_limit_ms=limit)
    print(f"{q.name}: |E|={len(q.edges)} labels={[int(q.labels[u]) for u in order]} bw={bw} "
          f"aut={inf.get('automorphisms')} count={c} dfs_ms={st['dfs_ms']:.1f} tasks={st['tasks']} "
          f"words={st['words']} pool={st['pool_size']}@{st['pool_depth']} timed_out={st['timed_out']}",
          flush=True)

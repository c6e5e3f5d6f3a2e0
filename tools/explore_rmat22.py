"""rmat22 small patterns (BASELINE config 3): count, time, tasks, idle rate per pattern.

    python tools/explore_rmat22.py [LIMIT_MS] [PATTERNS...]      (GM_LIB selects a library variant)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import gminputs as gi  # noqa: E402
import paper_2604_10601_b200 as gm  # noqa: E402

lim = float(sys.argv[1]) if len(sys.argv) > 1 else 20000.0
names = sys.argv[2:] or ["triangle", "clique4", "cycle5"]
cfg = bench.CONFIGS["rmat22"]
n, s, d, lab = bench.make_graph_device(cfg)
g = gm.gm_load_graph(n, s, d, lab, cfg["labels"])
mk = {"triangle": gi.triangle, "clique4": lambda: gi.clique(4), "clique5": lambda: gi.clique(5),
      "cycle4": lambda: gi.cycle(4), "cycle5": lambda: gi.cycle(5), "cycle6": lambda: gi.cycle(6)}
for name in names:
    q = mk[name]()
    p = gm.gm_plan_query(g, q)
    for it in range(2):
        c, st = gm.gm_count(p, time_limit_ms=lim, root_seed=int(os.environ.get("GM_ROOT_SEED", "1")),
                            symmetry=os.environ.get("GM_NOSYM") is None)
        idle = 1 - st["tasks"] / max(1, 32 * st["rounds"])
        print(json.dumps({"q": name, "count": c, "ms": round(st["total_ms"], 2), "dfs_ms": round(st["dfs_ms"], 2),
                          "timed_out": st["timed_out"], "tasks": st["tasks"], "words": st["words"],
                          "idle": round(idle, 4), "aut": st["automorphisms"], "pool": st["pool_size"],
                          "depth": st["pool_depth"], "order": p.info()["order"]}), flush=True)

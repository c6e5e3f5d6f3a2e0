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
                            symmetry=os.environ.get("GM_NOSYM") is None,
                            gen_cache=os.environ.get("GM_GEN_CACHE", "1") == "1")
        idle = 1 - st["tasks"] / max(1, 32 * st["rounds"])
        print(json.dumps({"q": name, "count": c, "ms": round(st["total_ms"], 2), "dfs_ms": round(st["dfs_ms"], 2),
                          "timed_out": st["timed_out"], "tasks": st["tasks"], "words": st["words"],
                          "idle": round(idle, 4), "aut": st["automorphisms"], "pool": st["pool_size"],
                          "depth": st["pool_depth"], "order": p.info()["order"]}), flush=True)

# GM_SAMPLE=f: also estimate each pattern's total from a uniform sample of a fraction f of its
# root candidates (root-restricted counts run without symmetry breaking)
frac = float(os.environ.get("GM_SAMPLE", "0"))
if frac > 0:
    import numpy as np
    for name in names:
        q = mk[name]()
        p = gm.gm_plan_query(g, q)
        u0 = p.info()["order"][0]
        cands = np.flatnonzero(p.candidates(u0))
        k = max(1, int(len(cands) * frac))
        roots = np.random.default_rng(7).permutation(cands)[:k].astype(np.uint32)
        c, st = gm.gm_count(p, roots=roots, time_limit_ms=60000.0)
        print(json.dumps({"q": name, "sample_roots": k, "of": int(len(cands)), "count": c,
                          "est_total": c * len(cands) / k, "ms": round(st["total_ms"], 2),
                          "timed_out": st["timed_out"], "tasks": st["tasks"]}), flush=True)

"""Explore which query sets complete on a bench graph: per-query count, ms, timed_out.

    python tools/explore_queries.py --config rmat18 --sizes 8 10 12 16 --seeds 1000 1001 1002 1003 --limit-ms 10000
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="rmat18")
    ap.add_argument("--sizes", type=int, nargs="+", default=[8, 12, 16])
    ap.add_argument("--seeds", type=int, nargs="+", default=[1000, 1001, 1002, 1003])
    ap.add_argument("--kinds", nargs="+", default=["dense"])
    ap.add_argument("--limit-ms", type=float, default=10000.0)
    ap.add_argument("--root-seed", type=int, default=0)
    args = ap.parse_args()
    import torch
    import bench
    import gminputs as gi
    import paper_2604_10601_b200 as gm
    cfg = bench.CONFIGS[args.config]
    n, s, d, lab = bench.make_graph_device(cfg)
    lh = lab.cpu().numpy().view(np.uint32)
    if cfg["scale"] <= 20:
        adj = gi.HostAdjacency(*gi.simple_adjacency(n, s.cpu().numpy().view(np.uint32), d.cpu().numpy().view(np.uint32)))
    else:
        import gminputs.gpu as gg
        adj = gg.DeviceNeighbors(n, s, d)
    g = gm.gm_load_graph(n, s, d, lab, cfg["labels"])
    for kind in args.kinds:
        for k in args.sizes:
            for sd in args.seeds:
                if kind == "dense":
                    q = gi.grow_query(adj, lh, k, seed=sd, dense=True, min_avg_degree=3.0)
                elif kind == "plain":
                    q = gi.grow_query(adj, lh, k, seed=sd)
                else:
                    q = gi.walk_query(adj, lh, k, seed=sd)
                p = gm.gm_plan_query(g, q)
                c, st = gm.gm_count(p, time_limit_ms=args.limit_ms, root_seed=args.root_seed)
                idle = 1 - st["tasks"] / max(1, 32 * st["rounds"])
                print(json.dumps({"kind": kind, "k": k, "seed": sd, "m": len(q.edges), "count": c,
                                  "ms": round(st["total_ms"], 2), "dfs_ms": round(st["dfs_ms"], 2),
                                  "timed_out": st["timed_out"], "tasks": st["tasks"], "idle": round(idle, 4),
                                  "aut": st["automorphisms"], "paths": st["paths"]}), flush=True)


if __name__ == "__main__":
    main()

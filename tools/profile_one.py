"""One DFS launch of a bench workload for ncu (no time limit: work bounded by a root sample).
   python tools/profile_one.py QUERY_INDEX NROOTS [CONFIG] [TAU]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import gminputs as gi  # noqa: E402
import paper_2604_10601_b200 as gm  # noqa: E402

qi = int(sys.argv[1]) if len(sys.argv) > 1 else 1
nroots = int(sys.argv[2]) if len(sys.argv) > 2 else 64
cfgname = sys.argv[3] if len(sys.argv) > 3 else "rmat18"
tau = int(float(sys.argv[4])) if len(sys.argv) > 4 else 1000000
cfg = bench.CONFIGS[cfgname]
n, s, d, lab = bench.make_graph_device(cfg)
lh = lab.cpu().numpy().view(np.uint32)
if cfg.get("dense") or cfg.get("sparse"):
    import gminputs.gpu as gg
    adj = gg.DeviceNeighbors(n, s, d)
else:
    adj = None                      # fixed patterns only
# query growth on scale-24/26 graphs scans the device edge list per vertex: cache the queries
import hashlib  # noqa: E402
cache = f"/tmp/gm_queries_{cfgname}_{hashlib.sha1(repr(sorted(cfg.items())).encode()).hexdigest()[:10]}.json"
if os.path.exists(cache):
    import json
    qs = [gi.Query(d_["n"], d_["edges"], d_["labels"], d_["name"]) for d_ in json.load(open(cache))]
else:
    qs = bench.build_queries(cfg, adj, lh)
    import json
    json.dump([{"n": int(q.n), "edges": q.edges.tolist(), "labels": q.labels.tolist(), "name": q.name} for q in qs],
              open(cache, "w"))
g = gm.gm_load_graph(n, s, d, lab, cfg["labels"])
if os.environ.get("GM_HUB_MB"):                 # hub-index sweeps
    g.build_hubs(int(float(os.environ["GM_HUB_MB"]) * (1 << 20)), int(os.environ.get("GM_HUB_MIN", "64")),
                 int(os.environ.get("GM_HUB_SUMM", "-1")))
q = qs[qi]
p = gm.gm_plan_query(g, q, filter=os.environ.get("GM_FILTER", "nlf"))
u0 = p.info()["order"][0]
cands = np.flatnonzero(p.candidates(u0))
roots = np.random.default_rng(0).permutation(cands)[:nroots].astype(np.uint32) if nroots > 0 else None
for it in range(2):
    t = time.time()
    c, st = gm.gm_count(p, roots=roots, tau=tau, time_limit_ms=float(os.environ.get("GM_LIMIT_MS", "0")),
                        warps_per_block=int(os.environ.get("GM_WPB", "0")),
                        blocks_per_sm=int(os.environ.get("GM_BPS", "0")),
                        root_seed=int(os.environ.get("GM_ROOT_SEED", "0")),
                        count_words=os.environ.get("GM_COUNT_WORDS", "0") == "1",
                        gen_cache=os.environ.get("GM_GEN_CACHE", "1") == "1")
    print(q.name, len(q.edges), c, f"wall {time.time() - t:.3f}s",
          {k: st[k] for k in ("dfs_ms", "total_ms", "tasks", "words", "pool_size", "pool_depth", "donations",
                              "grid", "block")}, flush=True)

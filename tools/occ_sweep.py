"""Occupancy sensitivity of the DRAM-bound configs: tasks done in a fixed time limit per query
at several resident-block counts (blocks_per_sm), one graph build.
   python tools/occ_sweep.py CONFIG LIMIT_MS BPS..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2604_10601_b200 as gm  # noqa: E402

cfgname = sys.argv[1]
limit = float(sys.argv[2])
bps_list = [int(x) for x in sys.argv[3:]] or [0]
cfg = bench.CONFIGS[cfgname]
n, s, d, lab = bench.make_graph_device(cfg)
lh = lab.cpu().numpy().view(np.uint32)
import gminputs.gpu as gg  # noqa: E402
qs = bench.build_queries(cfg, gg.DeviceNeighbors(n, s, d), lh)
g = gm.gm_load_graph(n, s, d, lab, cfg["labels"])
for q in qs:
    p = gm.gm_plan_query(g, q, filter="nlf")
    for bps in bps_list:
        for it in range(2):
            c, st = gm.gm_count(p, time_limit_ms=limit, blocks_per_sm=bps, root_seed=1)
        print(f"{q.name} bps={bps} grid={st['grid']} levels={st['stack_levels']} dfs_ms={st['dfs_ms']:.1f} "
              f"tasks={st['tasks']} tasks/s={st['tasks'] / st['dfs_ms'] * 1e3:.3e}", flush=True)

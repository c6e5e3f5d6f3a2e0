"""Time gm_load_graph from host (pinned and pageable) and device edge lists, repeated."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_10601_b200 as gm  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "rmat18"]
n, s, d, lab = bench.make_graph_device(cfg)
sh, dh, lh = (x.cpu().numpy().view(np.uint32) for x in (s, d, lab))
sp, dp, lp = (torch.from_numpy(x.view(np.int32)).pin_memory().numpy().view(np.uint32) for x in (sh, dh, lh))
for name, args in (("device", (s, d, lab)), ("pinned", (sp, dp, lp)), ("pageable", (sh, dh, lh))):
    for it in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        g = gm.gm_load_graph(n, *args, cfg["labels"])
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        t = time.perf_counter()
        g.free()
        torch.cuda.synchronize()
        print(f"{name} load {1e3 * dt:.1f} ms, free {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)

#!/bin/bash
# Parameter sweeps on dense (0,1,3 with 100 roots) and sparse (5, 300 ms limit) bench queries.
run() { echo "== $*"; for qi in 0 1 3; do env "$@" timeout 120 python tools/profile_one.py $qi 100 2>&1 | tail -1 | cut -c1-90; done;
        env "$@" GM_LIMIT_MS=300 timeout 120 python tools/profile_one.py 5 0 2>&1 | tail -1 | cut -c1-90; }
run GM_WPB=4
run GM_WPB=2
run GM_WPB=8
run GM_HUB_MB=32
run GM_HUB_MB=96
run GM_HUB_MB=64 GM_HUB_MIN=16
run GM_HUB_MB=0

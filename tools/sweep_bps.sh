#!/bin/bash
# blocks/SM x warps/block sweep on dense queries 0-3 (100 roots) and sparse 5 (300 ms)
for cfg in "GM_BPS=9 GM_WPB=4" "GM_BPS=7 GM_WPB=4" "GM_BPS=6 GM_WPB=4" "GM_BPS=5 GM_WPB=4" "GM_BPS=4 GM_WPB=4" "GM_BPS=3 GM_WPB=8"; do
  echo "== $cfg"
  for qi in 0 1 2 3; do env $cfg timeout 120 python tools/profile_one.py $qi 100 2>&1 | tail -1 | cut -c1-100; done
  env $cfg GM_LIMIT_MS=300 timeout 120 python tools/profile_one.py 5 0 2>&1 | tail -1 | cut -c1-130
done

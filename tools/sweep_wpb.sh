#!/bin/bash
# warps/block sweep (blocks/SM from occupancy) on dense queries 0-3 (100 roots) and sparse 5 (300 ms)
for w in 4 2 8; do
  echo "== GM_WPB=$w"
  for qi in 0 1 2 3; do GM_WPB=$w timeout 120 python tools/profile_one.py $qi 100 2>&1 | tail -1 | cut -c1-100; done
  GM_WPB=$w GM_LIMIT_MS=300 timeout 120 python tools/profile_one.py 5 0 2>&1 | tail -1 | cut -c1-130
done

#!/bin/bash
# Same-box A/B of several libgmatch builds on the dense bench queries (100 sampled roots)
# and one time-limited sparse query:  tools/ab_multi.sh LIB... ("" = the in-tree build)
for qi in 0 1 2 3; do
  for lib in "$@"; do
    GM_LIB=$lib timeout 120 python tools/profile_one.py $qi 100 2>&1 | tail -1 | cut -c1-120 | sed "s|^|[${lib:-cur}] |"
  done
done
for lib in "$@"; do
  GM_LIB=$lib GM_LIMIT_MS=300 timeout 120 python tools/profile_one.py 5 0 2>&1 | tail -1 | cut -c1-120 | sed "s|^|[${lib:-cur}] |"
done

#!/bin/bash
# hub-index budget sweep on a large config: tools/sweep_hub.sh CONFIG NROOTS "QUERY..." "MB..."
CFG=$1; NR=$2; QS=$3; MBS=$4
for mb in $MBS; do
  echo "== GM_HUB_MB=$mb"
  for qi in $QS; do GM_HUB_MB=$mb GM_LIMIT_MS=1000 timeout 300 python tools/profile_one.py $qi $NR $CFG 2>&1 | tail -1 | cut -c1-150; done
done

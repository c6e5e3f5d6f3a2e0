#!/bin/bash
# Same-box A/B on one config: tools/ab_cfg.sh CONFIG NROOTS "QUERY..." LIB... ("" = in-tree build)
CFG=$1; NR=$2; QS=$3; shift 3
for qi in $QS; do
  for lib in "$@"; do
    GM_LIB=$lib timeout 300 python tools/profile_one.py $qi $NR $CFG 2>&1 | tail -1 | cut -c1-140 | sed "s|^|[${lib:-cur}] |"
  done
done

#!/bin/bash
# A/B timing of two libgmatch builds on the same box: tools/ab.sh <libA> <query...>
A=$1; shift
for qi in "$@"; do
  for lib in "$A" ""; do
    GM_LIB=$lib timeout 120 python tools/profile_one.py $qi 100 2>&1 | tail -1 | cut -c1-110 | sed "s|^|[${lib:-B}] |"
  done
done

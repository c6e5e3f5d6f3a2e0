#!/bin/bash
# Round-2 same-box A/B: build variants, then time each on rmat24 (all roots, 1 s limit: tasks
# done), rmat18 pair-counting queries (300 ms limit) and rmat18 dense queries (100 roots).
#   tools/ab_r2.sh OUTDIR  "name:flags" ...      ("cur:" = the in-tree build)
OUT=$1; shift
mkdir -p $OUT
LIBS=()
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  if [ "$name" = cur ]; then LIBS+=(""); continue; fi
  case $flags in *.so) LIBS+=("$flags"); continue ;; esac     # a prebuilt library
  tools/build_variant.sh /tmp/gm_$name.so paper_2604_10601_b200/csrc $flags && LIBS+=(/tmp/gm_$name.so)
done
run() {  # cfg nroots limit qi...
  local cfg=$1 nr=$2 lim=$3; shift 3
  for qi in "$@"; do
    for lib in "${LIBS[@]}"; do
      GM_LIB=$lib GM_LIMIT_MS=$lim timeout 300 python tools/profile_one.py $qi $nr $cfg 2>&1 | tail -1 | cut -c1-200 | sed "s|^|[${lib:-cur}] $cfg q$qi |"
    done
  done
}
SETS=${AB_SETS:-"pair dense r24"}
for set in $SETS; do
  case $set in
    pair)  run rmat18 0 300 4 5 6 7 > $OUT/ab_rmat18_pair.log 2>&1 ;;
    dense) run rmat18 100 0 0 1 2 3 > $OUT/ab_rmat18_dense.log 2>&1 ;;
    r24)   run rmat24 0 1000 0 1 2 3 > $OUT/ab_rmat24.log 2>&1 ;;
    r26)   run rmat26 0 1000 0 1 2 3 > $OUT/ab_rmat26.log 2>&1 ;;
    r22)   for lib in "${LIBS[@]}"; do
             GM_LIB=$lib timeout 300 python tools/explore_rmat22.py 5000 triangle clique4 cycle5 2>&1 | grep '^{' | sed "s|^|[${lib:-cur}] |"
           done > $OUT/ab_rmat22.log 2>&1 ;;
  esac
done

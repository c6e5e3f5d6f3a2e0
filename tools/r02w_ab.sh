# Lean stack A/B: cur = levels per query + AUXW rows + packed levels + per-query block size
# (up to 14 warps); v3 = same with 4-warp blocks; v2 = v3 without packing; head = round-2 HEAD.
O=gpurun_out/r02w; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $O/gputest.log 2>&1; echo "gputest rc $?" >> $O/gputest.log
tail -3 $O/gputest.log
for c in rmat24 rmat26; do
  for v in cur v3 v2 head; do
    case $v in cur) L="";; *) L=abl/gm_$v.so;; esac
    GM_LIB=$L GM_DEBUG_LAUNCH=1 timeout 600 python tools/occ_sweep.py $c 1000 0 > $O/occ_${c}_$v.log 2>&1
  done
done
AB_SETS="dense pair" tools/ab_r2.sh $O head:abl/gm_head.so cur:
for f in $O/occ_*.log $O/ab_*.log; do echo "== $f"; grep -v "^\[gm\]" $f | cut -c1-160; grep "^\[gm\]" $f | sort | uniq -c | head -8; done

# Lean stack (levels allocated per query) vs HEAD: GPU tests, then same-box A/B on rmat24/26/18.
O=gpurun_out/r02v; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $O/gputest.log 2>&1; echo "gputest rc $?" >> $O/gputest.log
tail -3 $O/gputest.log
for c in rmat24 rmat26; do
  GM_DEBUG_LAUNCH=1 timeout 600 python tools/occ_sweep.py $c 1000 0 > $O/occ_${c}_cur.log 2>&1
  GM_LIB=abl/gm_head.so GM_DEBUG_LAUNCH=1 timeout 600 python tools/occ_sweep.py $c 1000 0 > $O/occ_${c}_head.log 2>&1
done
GM_DEBUG_LAUNCH=1 timeout 600 python tools/occ_sweep.py rmat24 1000 4 5 > $O/occ_rmat24_bps.log 2>&1
AB_SETS="dense pair" tools/ab_r2.sh $O head:abl/gm_head.so cur:
for f in $O/occ_*.log $O/ab_*.log; do echo "== $f"; grep -v "^\[gm\]" $f | cut -c1-160; grep "^\[gm\]" $f | sort | uniq -c | head -8; done

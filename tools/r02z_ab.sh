# Parent lane packed into the vertex word of the 16/24/32-level stacks (GM_PACK_PID, in-tree)
# vs the lean-stack HEAD (abl/gm_v4.so): rmat26/24 A/B, then the GPU tests.
O=gpurun_out/r02z; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for c in rmat26 rmat24; do
  for v in cur v4; do
    case $v in cur) L="";; *) L=abl/gm_$v.so;; esac
    GM_LIB=$L GM_DEBUG_LAUNCH=1 timeout 600 python tools/occ_sweep.py $c 1000 0 > $O/occ_${c}_$v.log 2>&1
  done
done
timeout 1500 python -m pytest tests -x -q -m gpu > $O/gputest.log 2>&1; echo "gputest rc $?" >> $O/gputest.log
tail -3 $O/gputest.log
for f in $O/occ_*.log; do echo "== $f"; grep -v "^\[gm\]" $f | grep tasks; grep "^\[gm\]" $f | sort | uniq -c | cut -c1-150; done

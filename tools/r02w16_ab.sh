# 64-register deep kernels with blocks of up to 16 warps (32 warps per SM) vs HEAD (abl/gm_head2.so).
O=gpurun_out/r02w16; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for v in cur head2; do
  case $v in cur) L="";; *) L=abl/gm_$v.so;; esac
  GM_LIB=$L GM_DEBUG_LAUNCH=1 timeout 600 python tools/occ_sweep.py rmat24 1000 0 > $O/occ_rmat24_$v.log 2>&1
done
timeout 1200 python -m pytest tests -x -q -m gpu > $O/gputest.log 2>&1; echo "gputest rc $?" >> $O/gputest.log
tail -3 $O/gputest.log
for f in $O/occ_*.log; do echo "== $f"; grep -v "^\[gm\]" $f | grep tasks; grep "^\[gm\]" $f | sort | uniq -c | cut -c1-150; done

python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
tools/build_variant.sh /tmp/gm_prev.so abl/prev/paper_2604_10601_b200/csrc
AB_SETS="dense pair r22 r24 r26" tools/ab_r2.sh gpurun_out/r02k cur: loop8:-DGM_WIDE_LOOP8=1 hubfirst:-DGM_CHK_HUBFIRST=1 prev:/tmp/gm_prev.so
cat gpurun_out/r02k/*.log | cut -c1-170

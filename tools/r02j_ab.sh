python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
tools/build_variant.sh /tmp/gm_prev.so abl/prev/paper_2604_10601_b200/csrc
AB_SETS="dense pair r22 r24" tools/ab_r2.sh gpurun_out/r02j cur: prev:/tmp/gm_prev.so
cat gpurun_out/r02j/*.log | cut -c1-180

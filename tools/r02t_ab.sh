python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
tools/build_variant.sh /tmp/gm_pf.so paper_2604_10601_b200/csrc -DGM_PREFETCH_ROWS=1
AB_SETS="dense pair r24" tools/ab_r2.sh gpurun_out/r02t cur: pf:/tmp/gm_pf.so
cat gpurun_out/r02t/*.log | cut -c1-130

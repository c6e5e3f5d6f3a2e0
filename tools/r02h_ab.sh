python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
AB_SETS="dense pair r24 r22" tools/ab_r2.sh gpurun_out/r02h cur: wt4:-DGM_WIDE_T=4 w16:-DGM_WIDE_T16=4
cat gpurun_out/r02h/*.log | cut -c1-180

python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
AB_SETS="r22 dense pair r24" tools/ab_r2.sh gpurun_out/r02d cur: nocut:-DGM_CUT_MIN=0 nowords:-DGM_WORDS=0
cat gpurun_out/r02d/*.log | cut -c1-230

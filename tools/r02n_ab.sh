python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
AB_SETS="dense r24" tools/ab_r2.sh gpurun_out/r02n cur: nopair:-DGM_PAIR_CODE=0
cat gpurun_out/r02n/*.log | cut -c1-130

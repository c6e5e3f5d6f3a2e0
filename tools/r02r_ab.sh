python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
AB_SETS="r24 r26" tools/ab_r2.sh gpurun_out/r02r cur: nosumm:-DGM_HUB_SUMMARY=0 minb6:-DGM_MINB16=6 unroll16:-DGM_WIDE_LOOP16=0
cat gpurun_out/r02r/*.log | cut -c1-130

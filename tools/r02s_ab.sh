python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
AB_SETS="dense pair r24" tools/ab_r2.sh gpurun_out/r02s cur: noteam:-DGM_TEAM_CODE=0 novhub:-DGM_VHUB=0
cat gpurun_out/r02s/*.log | cut -c1-130

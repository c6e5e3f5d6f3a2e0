python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
AB_SETS="pair" tools/ab_r2.sh gpurun_out/r02q cur: vec8:-DGM_TWO_VEC8=1
cat gpurun_out/r02q/*.log | cut -c1-130

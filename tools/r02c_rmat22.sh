mkdir -p gpurun_out/r02c
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02c/build.log 2>&1
tools/build_variant.sh /tmp/gm_lvl.so paper_2604_10601_b200/csrc -DGM_LEVEL_STATS
timeout 600 python tools/explore_rmat22.py 20000 triangle clique4 cycle5 > gpurun_out/r02c/rmat22_cur.log 2>&1
GM_LIB=/tmp/gm_lvl.so timeout 600 python tools/explore_rmat22.py 20000 clique4 cycle5 > gpurun_out/r02c/rmat22_lvl.log 2>&1
GM_SAMPLE=0.002 timeout 900 python tools/explore_rmat22.py 1 cycle5 clique4 > gpurun_out/r02c/rmat22_sample.log 2>&1
cat gpurun_out/r02c/*.log | grep -v "^\[gm\]" | cut -c1-400

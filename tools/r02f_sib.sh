mkdir -p gpurun_out/r02f
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02f/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "sibling or clique or symmetry or count_random" > gpurun_out/r02f/sibtest.log 2>&1; echo "rc $?" >> gpurun_out/r02f/sibtest.log
tail -15 gpurun_out/r02f/sibtest.log
tools/build_variant.sh /tmp/gm_nosib.so paper_2604_10601_b200/csrc -DGM_SIB=0
for lib in "" /tmp/gm_nosib.so; do GM_LIB=$lib timeout 300 python tools/explore_rmat22.py 5000 clique4 triangle 2>&1 | grep '^{' | cut -c1-200 | sed "s|^|[${lib:-cur}] |"; done

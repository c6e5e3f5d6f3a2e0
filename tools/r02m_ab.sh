python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "generate_cache or sibling or count_random or symmetry" > gpurun_out/r02m_tests.log 2>&1; echo "rc $?" >> gpurun_out/r02m_tests.log; tail -3 gpurun_out/r02m_tests.log
AB_SETS="r22 dense pair r24" tools/ab_r2.sh gpurun_out/r02m cur: nogen:-DGM_GEN_CACHE=0 tsib4:-DGM_WIDE_TSIB=4
cat gpurun_out/r02m/*.log | cut -c1-150

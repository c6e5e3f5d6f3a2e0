python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large_queries.py -x -q -m gpu > gpurun_out/r02l_tests.log 2>&1; echo "rc $?" >> gpurun_out/r02l_tests.log; tail -3 gpurun_out/r02l_tests.log
AB_SETS="dense pair r22 r24" tools/ab_r2.sh gpurun_out/r02l cur: nogen:-DGM_GEN_CACHE=0
cat gpurun_out/r02l/*.log | cut -c1-150

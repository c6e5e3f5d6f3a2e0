python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r02p_tests.log 2>&1; echo "rc $?" >> gpurun_out/r02p_tests.log; tail -3 gpurun_out/r02p_tests.log
tools/build_variant.sh /tmp/gm_prev3.so abl/prev3/paper_2604_10601_b200/csrc
AB_SETS="dense pair r22 r26" tools/ab_r2.sh gpurun_out/r02p cur: prev3:/tmp/gm_prev3.so
cat gpurun_out/r02p/*.log | cut -c1-130

mkdir -p gpurun_out/r02b
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02b/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r02b/gputest.log 2>&1; echo "gputest rc $?" >> gpurun_out/r02b/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b/smoke.log 2>&1
timeout 900 python bench.py --per-query > gpurun_out/r02b/bench.json 2> gpurun_out/r02b/bench.err
tail -3 gpurun_out/r02b/gputest.log; cat gpurun_out/r02b/smoke.log; cat gpurun_out/r02b/bench.json

# Round-2 re-entry check: HEAD builds, GPU tests, smoke, default bench.
O=gpurun_out/r02u; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $O/gputest.log 2>&1; echo "gputest rc $?" >> $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python bench.py > $O/bench_rmat18.json 2> $O/bench_rmat18.err
tail -3 $O/gputest.log; cat $O/smoke.log; cat $O/bench_rmat18.json | cut -c1-600

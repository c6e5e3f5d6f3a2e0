# Final HEAD check: GPU tests, smoke, the 2-rank bench path, and an ncu capture of a rmat26 32-vertex query.
O=gpurun_out/r02y; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $O/gputest.log 2>&1; echo "gputest rc $?" >> $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
GM_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 1 --warmup 3 --no-context --no-cpu-baseline > $O/bench_2rank.json 2> $O/bench_2rank.err
GM_LIMIT_MS=300 GM_DEBUG_LAUNCH=1 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_dfs -c 1 -f -o $O/k_dfs_rmat26_rq32_s1003 python tools/profile_one.py 3 0 rmat26 > $O/ncu26.log 2>&1
python tools/ncu_summary.py $O/k_dfs_rmat26_rq32_s1003.ncu-rep > $O/k_dfs_rmat26_rq32_s1003.md 2>&1
python tools/ncu_lines.py $O/k_dfs_rmat26_rq32_s1003.ncu-rep > $O/k_dfs_rmat26_rq32_s1003_lines.md 2>&1
tail -3 $O/gputest.log; cat $O/smoke.log; cut -c1-300 $O/bench_2rank.json; head -22 $O/k_dfs_rmat26_rq32_s1003.md

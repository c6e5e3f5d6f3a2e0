# Round-2 final session, part 2 (after the hub-summary compile-out): tests, rmat24/26 benches, rmat24 ncu capture
set -x
O=gpurun_out/r02final2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $O/gputest.log 2>&1; echo "gputest rc $?" >> $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
for c in rmat24 rmat26; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-context > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --config rmat24 --steps 2 --warmup 3 --no-cpu-baseline --no-context --root-order hubs > $O/bench_rmat24_hubs.json 2> $O/bench_rmat24_hubs.err
GM_LIMIT_MS=300 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dfs -c 1 -f -o $O/k_dfs_rmat24_rq1000 python tools/profile_one.py 0 0 rmat24 > $O/ncu24.log 2>&1
python tools/ncu_summary.py $O/k_dfs_rmat24_rq1000.ncu-rep > $O/k_dfs_rmat24_rq1000.md 2>&1
tail -3 $O/gputest.log; cat $O/smoke.log; ls -la $O

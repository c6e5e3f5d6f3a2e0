# Round-2 final measurement session: tests, smoke, benches, ncu launch list + full captures.
set -x
O=gpurun_out/r02final; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $O/gputest.log 2>&1; echo "gputest rc $?" >> $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python bench.py > $O/bench_rmat18.json 2> $O/bench_rmat18.err
for c in rmat22 rmat24 rmat26; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-context > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --config rmat24 --steps 2 --warmup 3 --no-cpu-baseline --no-context --root-order hubs > $O/bench_rmat24_hubs.json 2> $O/bench_rmat24_hubs.err
# the multi-rank path end to end: 2 ranks time-slicing one GPU (gloo for the host collectives)
GM_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 1 --warmup 3 --no-context --no-cpu-baseline > $O/bench_2rank.json 2> $O/bench_2rank.err
# launch list of a short bench run (the same command, fewer steps; under ncu every launch is serialised)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_rmat18.csv \
  python bench.py --steps 1 --warmup 3 --no-context --no-cpu-baseline > $O/launches_bench.log 2>&1
# full captures: the bench's first k_dfs launch (rq8_s1000, shuffled roots, 1 s), rmat24 rq16_s1000 (300 ms), rmat22 4-clique (300 ms)
GM_LIMIT_MS=1000 GM_ROOT_SEED=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dfs -c 1 -f -o $O/k_dfs_rmat18_rq1000 python tools/profile_one.py 0 0 rmat18 > $O/ncu18.log 2>&1
GM_LIMIT_MS=300 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dfs -c 1 -f -o $O/k_dfs_rmat24_rq1000 python tools/profile_one.py 0 0 rmat24 > $O/ncu24.log 2>&1
GM_LIMIT_MS=300 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dfs -c 1 -f -o $O/k_dfs_rmat22_clique4 python tools/profile_one.py 1 0 rmat22 > $O/ncu22.log 2>&1
for r in $O/*.ncu-rep; do python tools/ncu_summary.py $r > ${r%.ncu-rep}.md 2>&1; done
python tools/ncu_summary.py $O/launches_rmat18.csv > $O/launches_rmat18.md 2>&1
tail -3 $O/gputest.log; cat $O/smoke.log; ls -la $O

# Round-2 final measurements of the lean-stack build: smoke, benches, ncu launch list and full captures.
O=gpurun_out/r02x; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python bench.py > $O/bench_rmat18.json 2> $O/bench_rmat18.err
for c in rmat24 rmat26 rmat22; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-context > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --config rmat24 --steps 2 --warmup 3 --no-cpu-baseline --no-context --root-order hubs > $O/bench_rmat24_hubs.json 2> $O/bench_rmat24_hubs.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_rmat18.csv \
  python bench.py --steps 1 --warmup 3 --no-context --no-cpu-baseline > $O/launches_bench.log 2>&1
GM_LIMIT_MS=1000 GM_ROOT_SEED=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dfs -c 1 -f -o $O/k_dfs_rmat18_rq1000 python tools/profile_one.py 0 0 rmat18 > $O/ncu18.log 2>&1
GM_LIMIT_MS=300 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dfs -c 1 -f -o $O/k_dfs_rmat24_rq1000 python tools/profile_one.py 0 0 rmat24 > $O/ncu24.log 2>&1
for r in $O/*.ncu-rep; do python tools/ncu_summary.py $r > ${r%.ncu-rep}.md 2>&1; done
python tools/ncu_summary.py $O/launches_rmat18.csv > $O/launches_rmat18.md 2>&1
cat $O/smoke.log; for f in $O/bench_*.json; do echo "$f $(cut -c1-200 $f)"; done; ls -la $O

set -x
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
# filter / hub-budget experiments on rmat24 (every root, 1 s, tasks done)
for q in 0 1 3; do
  GM_LIMIT_MS=1000 timeout 300 python tools/profile_one.py $q 0 rmat24 2>&1 | tail -1 | cut -c1-200 | sed "s/^/[nlf] /"
  GM_FILTER=none GM_LIMIT_MS=1000 timeout 300 python tools/profile_one.py $q 0 rmat24 2>&1 | tail -1 | cut -c1-200 | sed "s/^/[none] /"
  GM_HUB_MB=32768 GM_LIMIT_MS=1000 timeout 300 python tools/profile_one.py $q 0 rmat24 2>&1 | tail -1 | cut -c1-200 | sed "s/^/[hub32g] /"
done > gpurun_out/r02/exp_rmat24_filter_hubs.log 2>&1
# ncu: launch list of one bench step
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/launches_rmat18.csv python bench.py --steps 1 --warmup 1 --no-context --no-cpu-baseline > gpurun_out/r02/launches_bench.log 2>&1
# ncu full: the bench's first k_dfs launch as the bench runs it (rq8_s1000, shuffled roots, 1 s limit)
GM_LIMIT_MS=1000 GM_ROOT_SEED=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dfs -c 1 -f -o gpurun_out/r02/k_dfs_rmat18_rq1000 python tools/profile_one.py 0 0 rmat18 > gpurun_out/r02/ncu1.log 2>&1
# ncu full: rmat24 rq16_s1000 (DRAM-bound), 300 ms
GM_LIMIT_MS=300 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dfs -c 1 -f -o gpurun_out/r02/k_dfs_rmat24_rq1000 python tools/profile_one.py 0 0 rmat24 > gpurun_out/r02/ncu2.log 2>&1
ls -la gpurun_out/r02

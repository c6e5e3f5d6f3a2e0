# round-2 ncu captures of the current build (each after the same command ran clean without ncu)
set -x
O=gpurun_out/r02i; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
GM_LIMIT_MS=1000 GM_ROOT_SEED=1 timeout 300 python tools/profile_one.py 0 0 rmat18 > $O/plain18.log 2>&1 && \
GM_LIMIT_MS=1000 GM_ROOT_SEED=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dfs -c 1 -f -o $O/k_dfs_rmat18_rq1000 python tools/profile_one.py 0 0 rmat18 > $O/ncu18.log 2>&1
GM_LIMIT_MS=300 timeout 300 python tools/profile_one.py 0 0 rmat24 > $O/plain24.log 2>&1 && \
GM_LIMIT_MS=300 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dfs -c 1 -f -o $O/k_dfs_rmat24_rq1000 python tools/profile_one.py 0 0 rmat24 > $O/ncu24.log 2>&1
GM_LIMIT_MS=300 timeout 300 python tools/profile_one.py 1 0 rmat22 > $O/plain22.log 2>&1 && \
GM_LIMIT_MS=300 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dfs -c 1 -f -o $O/k_dfs_rmat22_clique4 python tools/profile_one.py 1 0 rmat22 > $O/ncu22.log 2>&1
for r in $O/*.ncu-rep; do python tools/ncu_summary.py $r > ${r%.ncu-rep}.md 2>&1; done
ls -la $O; tail -2 $O/plain*.log

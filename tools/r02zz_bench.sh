# Final HEAD benches: smoke, rmat18 headline, rmat24, rmat26.
O=gpurun_out/r02zz; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python bench.py > $O/bench_rmat18.json 2> $O/bench_rmat18.err
for c in rmat26 rmat24; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-context > $O/bench_$c.json 2> $O/bench_$c.err
done
cat $O/smoke.log; for f in $O/bench_*.json; do echo "$f $(cut -c1-160 $f)"; done

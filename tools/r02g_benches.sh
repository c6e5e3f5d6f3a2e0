mkdir -p gpurun_out/r02g
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02g/build.log 2>&1
for c in rmat22 rmat24 rmat26; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-context > gpurun_out/r02g/bench_$c.json 2> gpurun_out/r02g/bench_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/r02g/bench_$c.json')); print('$c', {k: d[k] for k in ('value','ms_per_step','tasks_per_s','idle_rate')}, d['roofline']['frac']); [print('  ', r['q'], r['embeddings'], r['completed'], r['ms'], r['tasks'], r['D']) for r in d['per_query']]"
done
AB_SETS="dense r26" tools/ab_r2.sh gpurun_out/r02g cur: wt4:-DGM_WIDE_T=4 minb4:-DGM_MINB32=4
cat gpurun_out/r02g/ab_*.log | cut -c1-200

mkdir -p gpurun_out/r02e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02e/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r02e/gputest.log 2>&1; echo "gputest rc $?" >> gpurun_out/r02e/gputest.log
timeout 900 python bench.py > gpurun_out/r02e/bench.json 2> gpurun_out/r02e/bench.err
tail -3 gpurun_out/r02e/gputest.log; python -c "
import json; d=json.load(open('gpurun_out/r02e/bench.json')); print({k: d[k] for k in ('value','ms_per_step','tasks_per_s','idle_rate','gpu_launches')}); print(d['roofline']); print(d['e2e']); print([ (r['q'], r['embeddings'], r['ms'], r['tasks']) for r in d['per_query']]); print({k:(v['value'] if isinstance(v,dict) and 'value' in v else None) for k,v in d['context'].items()})"
tail -5 gpurun_out/r02e/bench.err

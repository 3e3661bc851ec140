set -e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
set +e
python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
python bench.py --steps 10 --warmup 3 --no-cpu --no-secondary > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 600 gpurun_out/bench.err
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], {k:(round(v['ms_per_step'],3)) for k,v in d['kernels'].items()}, d['kernels']['k_refine_hard']['queued_px_per_step'])"

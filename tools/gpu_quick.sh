# quick GPU check: build, matching/golden/baseline parity tests, headline bench breakdown
set +e
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_matching_gpu.py tests/test_golden.py tests/test_baseline_parity_gpu.py ${EXTRA_TESTS} -q -x -rA -m gpu > gpurun_out/t.log 2>&1; grep -E "passed|failed|Error|config2:" gpurun_out/t.log | tail -6
timeout 600 python bench.py --no-cpu --no-secondary --steps 10 > gpurun_out/bench.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print(round(d['value']/1e9,3), 'Gpx/s', round(d['ms_per_step'],3), 'ms'); print({k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['kernels']['k_match_refine'].get('exact_path_px_per_step'))" || tail -20 gpurun_out/bench.log

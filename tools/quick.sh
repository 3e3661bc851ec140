# quick GPU check: matching parity tests + headline bench breakdown
timeout 600 python -m pytest tests/test_matching_gpu.py tests/test_golden.py -q -x > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
timeout 600 python bench.py --no-cpu --no-secondary --steps 5 > gpurun_out/bench.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print(round(d['value']/1e9,3), 'Gpx/s', round(d['ms_per_step'],3), 'ms'); print({k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" || tail -20 gpurun_out/bench.log

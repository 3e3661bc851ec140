# GPU box pass: build, GPU tests (with timings), smoke, quick bench.
set +e
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt 2>&1; free -g > gpurun_out/free.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1; tail -25 gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --no-cpu --steps 10 > gpurun_out/bench.log 2>&1; tail -c 600 gpurun_out/bench.log

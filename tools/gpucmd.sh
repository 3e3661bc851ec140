set -e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
set +e
nproc > gpurun_out/host.txt; lscpu | grep "Model name" >> gpurun_out/host.txt
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; tail -1 gpurun_out/bench_full.log
python bench.py --steps 2 --warmup 3 --no-cpu --no-secondary > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-secondary > gpurun_out/ncu_launch.log 2>&1; tail -2 gpurun_out/ncu_launch.log

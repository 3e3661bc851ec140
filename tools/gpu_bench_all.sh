set +e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"; tail -c 400 gpurun_out/bench_full.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -c 300 gpurun_out/bench_ref.log
timeout 900 python bench.py --backend-sharded --no-cpu --no-secondary --steps 3 > gpurun_out/bench_sharded.log 2>&1; echo "sharded rc=$?"; tail -c 300 gpurun_out/bench_sharded.log

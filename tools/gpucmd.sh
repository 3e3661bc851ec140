set -e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
set +e
python -m pytest tests/test_backend_gpu.py tests/test_tracking_gpu.py tests/test_distributed.py -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
python tools/probe_backend.py --iters 4 > gpurun_out/pb.log 2>&1; tail -1 gpurun_out/pb.log

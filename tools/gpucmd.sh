set -e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
set +e
python -m pytest tests/test_matching_gpu.py -m gpu -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
python tools/probe_match.py --edges 8 --modes r0,r1,r3x1,refine --reps 3 > gpurun_out/probe.log 2>&1; cat gpurun_out/probe.log

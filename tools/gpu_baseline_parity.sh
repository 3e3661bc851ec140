set +e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_baseline_parity_gpu.py -q -x -rA -m gpu --durations=5 > gpurun_out/t.log 2>&1; grep -E "passed|failed|Error|config|assert|worst" gpurun_out/t.log | tail -30

python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/ -m gpu -q -x 2>&1 | tail -3
python tools/probe_backend.py 2>&1 | tail -4
python tools/probe_match.py --edges 8 2>&1 | tail -2

set -e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
set +e
timeout 900 python -m pytest tests/ -m gpu -q 2>&1 | tail -4
python tools/probe_backend.py 2>&1 | tail -2

set -e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
set +e
python tools/moved_tmp.py > gpurun_out/moved.log 2>&1; cat gpurun_out/moved.log | tail -5

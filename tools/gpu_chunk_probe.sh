set +e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for n in 4 8 16 64; do python tools/time_match.py $n 2>&1 | tail -1; done

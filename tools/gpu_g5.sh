set +e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv \
  python tools/ncu_target.py backend > gpurun_out/c3_ncu.log 2>&1; echo "rc=$?"

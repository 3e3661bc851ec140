set +e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python tools/ncu_target.py backend > gpurun_out/plain_backend.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_ldlt_sky' -s 1 -c 1 \
  -o gpurun_out/prof_sky -f python tools/ncu_target.py backend > gpurun_out/ncu_sky.log 2>&1; echo "ncu rc=$?"

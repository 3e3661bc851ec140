# Final GPU pass of the round: build, full GPU suite, smoke, ncu of the frontal solve (final code).
set +e
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/gpu_tests_final.log 2>&1; tail -4 gpurun_out/gpu_tests_final.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_final.log 2>&1; tail -1 gpurun_out/smoke_final.log
timeout 300 python tools/ncu_target.py backend > gpurun_out/plain_backend.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_ldlt_sky|k_sky_entries' -s 2 -c 2 \
  -o gpurun_out/prof_sky_final -f python tools/ncu_target.py backend > gpurun_out/ncu_sky_final.log 2>&1; echo "ncu rc=$?"

# time every build/variants/* library + the default build on the config-2 matcher
set +e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
python tools/time_match.py ${EDGES:-64} 2>&1 | tail -1
for d in build/variants/*/; do PMX_LIB=$d/libpmx_cuda.so python tools/time_match.py ${EDGES:-64} 2>&1 | tail -1; done

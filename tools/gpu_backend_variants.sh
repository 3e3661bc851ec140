set +e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for c in c3 ${EXTRA_CFG}; do
python tools/time_backend.py $c 2>&1 | tail -1
for d in build/variants/*/; do PMX_LIB=$d/libpmx_cuda.so python tools/time_backend.py $c 2>&1 | tail -1; done
done

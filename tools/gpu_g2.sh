set +e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
PMX_LIB=build/variants/skyt/libpmx_cuda.so timeout 300 python tools/time_backend.py c3 > gpurun_out/skyt.log 2>&1
grep "sky warp" gpurun_out/skyt.log | sort | uniq -c | sort -rn | head -12
tail -1 gpurun_out/skyt.log

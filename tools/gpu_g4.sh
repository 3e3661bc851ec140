set +e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
EXTRA_CFG=${EXTRA_CFG:-} bash tools/gpu_backend_variants.sh
timeout 900 python -m pytest tests -m gpu -q -x -k "${PYK:-backend or config3 or config4 or exactness or sharded}" > gpurun_out/t_backend.log 2>&1; tail -3 gpurun_out/t_backend.log

set +e
EXTRA_CFG=c4 bash tools/gpu_backend_variants.sh
timeout 900 python -m pytest tests -m gpu -q -x -k "backend or config3 or config4 or exactness or sharded" > gpurun_out/t_backend.log 2>&1; tail -3 gpurun_out/t_backend.log

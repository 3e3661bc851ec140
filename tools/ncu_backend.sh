set -e
python tools/ncu_target.py backend 100 > gpurun_out/plain_backend.log 2>&1
ncu --set full --clock-control none --import-source on -k 'regex:k_edge_terms_ray|k_ldlt_sky' -c 2 \
    -o gpurun_out/prof_be -f python tools/ncu_target.py backend 100 > gpurun_out/ncu_be.log 2>&1
echo done

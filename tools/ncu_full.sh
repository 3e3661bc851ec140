# Full ncu captures of the matching and backend kernels (run under gpurun).
set -e
python tools/ncu_target.py match 5 > gpurun_out/plain_match.log 2>&1
ncu --set full --clock-control none --import-source on -k 'regex:k_match_refine|k_prep' -c 3 \
    -o gpurun_out/prof_match -f python tools/ncu_target.py match 5 > gpurun_out/ncu_match.log 2>&1
python tools/ncu_target.py backend 100 > gpurun_out/plain_backend.log 2>&1
ncu --set full --clock-control none --import-source on -k 'regex:k_edge_terms_ray|k_ldlt_sky' -c 2 \
    -o gpurun_out/prof_backend -f python tools/ncu_target.py backend 100 > gpurun_out/ncu_backend.log 2>&1
echo done

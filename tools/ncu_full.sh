# Full ncu captures of the matching and backend kernels (run under gpurun).
set -e
python tools/ncu_target.py match 6 > gpurun_out/plain_match.log 2>&1
ncu --set full --clock-control none --import-source on -k 'regex:k_prep|k_match|k_refine_pairs|k_refine_hard|k_sel_hist' -c 6 \
    -o gpurun_out/prof_match -f python tools/ncu_target.py match 6 > gpurun_out/ncu_match.log 2>&1
python tools/ncu_target.py backend 100 > gpurun_out/plain_backend.log 2>&1
ncu --set full --clock-control none --import-source on -k 'regex:k_edge_terms_ray|k_ldlt' -c 3 \
    -o gpurun_out/prof_backend -f python tools/ncu_target.py backend 100 > gpurun_out/ncu_backend.log 2>&1
echo done

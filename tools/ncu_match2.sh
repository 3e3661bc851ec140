set -e
python tools/ncu_target.py match 5 > gpurun_out/plain_match.log 2>&1
ncu --set full --clock-control none --import-source on -k 'regex:k_refine_q8|k_match|k_prep' -c 3 \
    -o gpurun_out/prof_m2 -f python tools/ncu_target.py match 5 > gpurun_out/ncu_m2.log 2>&1
echo done

# ncu --set full of the fused matcher (source attribution), 5 config-2 edges.
set -e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python tools/ncu_target.py match 5 > gpurun_out/plain_match.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k 'regex:k_match_refine|k_prep' -s 2 -c 2 \
    -o gpurun_out/prof_match_r02 -f python tools/ncu_target.py match 5 > gpurun_out/ncu_match.log 2>&1
echo done

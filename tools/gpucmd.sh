python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python tools/probe_match.py --edges 8 --modes refine --reps 1 > gpurun_out/probe.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_match|k_refine_pairs" -c 2 -o gpurun_out/prof2 python tools/probe_match.py --edges 8 --reps 1 --modes refine > gpurun_out/ncu.log 2>&1; tail -2 gpurun_out/ncu.log

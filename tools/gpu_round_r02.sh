# Round-2 measurement pass: full bench (both arms), launch list of the
# headline command, one ncu --set full capture of the top kernel.
set +e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-secondary > gpurun_out/plain_headline.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-secondary \
  > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 300 python tools/ncu_target.py match 5 > gpurun_out/plain_match.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_match_refine' -s 1 -c 1 \
  -o gpurun_out/prof_match_r02b -f python tools/ncu_target.py match 5 > gpurun_out/ncu_match.log 2>&1; echo "full rc=$?"

# Targeted ncu metrics of every hot kernel (one ncu call; dram / lts bytes,
# issue, occupancy, pipes), then the per-kernel summary into gpurun_out/.
set -e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python tools/ncu_target.py all > gpurun_out/plain_all.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,l1tex__t_bytes.sum,\
sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed,\
smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,\
launch__registers_per_thread,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,\
smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,launch__grid_size
ncu --metrics $M --clock-control none \
    -k 'regex:k_prep|k_match_refine|k_sel_hist|k_track_gn|k_fuse|k_edge_terms_ray|k_ldlt_sky|k_bcr|k_cost64_ray|k_edge_blocks|k_sky_assemble|k_edge_sum_ray' \
    -c 120 --csv --log-file gpurun_out/ncu_all.csv python tools/ncu_target.py all > gpurun_out/ncu_all.log 2>&1
echo done

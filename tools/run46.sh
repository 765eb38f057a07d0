#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__t_bytes.sum,l1tex__t_sector_hit_rate.pct,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_elapsed,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_elapsed
timeout 900 ncu --graph-profiling graph --metrics $M --clock-control none --print-units base --csv --log-file gpurun_out/s5_solve_graph_final.csv python tools/solve_once.py > gpurun_out/s5_solve_graph_final.log 2>&1
echo "ncu graph rc=$?"; tail -n 2 gpurun_out/s5_solve_graph_final.log

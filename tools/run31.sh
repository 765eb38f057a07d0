#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
HDDM_NO_GRAPHS=1 timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_fp64.sum,smsp__thread_inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none --print-units base --csv --log-file gpurun_out/s5_solve_inst.csv python tools/solve_once.py > gpurun_out/s5_solve_inst.log 2>&1
echo rc=$?; tail -2 gpurun_out/s5_solve_inst.log

#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
HDDM_NO_GRAPHS=1 timeout 1500 ncu --section SourceCounters --section WarpStateStats --section LaunchStats --import-source on --clock-control none -k regex:'k_bwd_stage|k_fwd_pull$' --launch-skip 140 -c 140 -o gpurun_out/s5_hot -f python tools/solve_once.py > gpurun_out/s5_hot.log 2>&1
echo rc=$?; tail -2 gpurun_out/s5_hot.log; ls -la gpurun_out/s5_hot.ncu-rep

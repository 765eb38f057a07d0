#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_rhs_transfer|k_check|k_accumulate' -c 12 -o gpurun_out/s5_stages -f python tools/stage_prof.py > gpurun_out/s5_stages_ncu.log 2>&1
echo "ncu rc=$?"
ls -la gpurun_out/

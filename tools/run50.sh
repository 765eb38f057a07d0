#!/bin/bash
# ncu --set full of the staged backward pulls (one member group) and the member-tile forward pulls of a
# config-4 solve on the final kernels; summaries only (the reports are too large to bring back)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
HDDM_NO_GRAPHS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_bwd_stage' --launch-skip 44 -c 11 -o /tmp/s5_bwd_stage_full -f python tools/solve_once.py > gpurun_out/s5_bwd_stage_full.log 2>&1
echo "rc=$?"
HDDM_NO_GRAPHS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_fwd_pull' --launch-skip 232 -c 8 -o /tmp/s5_fwd_pull_full -f python tools/solve_once.py > gpurun_out/s5_fwd_pull_full.log 2>&1
echo "rc=$?"
for r in s5_bwd_stage_full s5_fwd_pull_full; do
ncu -i /tmp/$r.ncu-rep --page details --csv > gpurun_out/$r.details.csv 2>/dev/null
ncu -i /tmp/$r.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum,launch__grid_size,launch__registers_per_thread > gpurun_out/$r.raw.csv 2>/dev/null
done
ls -la gpurun_out/

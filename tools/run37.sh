#!/bin/bash
# session 5 final, part 1: ncu launch lists and step summaries of configs 4, 2, 3, 1 on the final kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 4 2 3 1; do
HDDM_NO_GRAPHS=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base --csv --log-file gpurun_out/final_launches_cfg$c.csv python bench.py --config $c --steps 3 --warmup 1 --skip-e2e --skip-cpu > gpurun_out/final_ncu$c.log 2>&1
echo "ncu cfg$c rc=$?"
python tools/ncu_step.py gpurun_out/final_launches_cfg$c.csv gpurun_out/final_step_summary_cfg$c.json | tail -3
done

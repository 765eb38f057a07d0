#!/bin/bash
cd $GRAFT_REPO_ROOT
for cfg in 4 3; do
for sr in 16 32 128 256 1000; do
HDDM_SPLIT_ROWS_MIN=$sr PCFG=$cfg TAG="cfg$cfg split_rows_min=$sr" python tools/time_step.py 2>&1 | grep RESULT
done
for sd in 12 24 96 200; do
HDDM_SPLIT_DIAG_MIN=$sd PCFG=$cfg TAG="cfg$cfg split_diag_min=$sd" python tools/time_step.py 2>&1 | grep RESULT
done
done

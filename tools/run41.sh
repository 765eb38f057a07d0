#!/bin/bash
cd $GRAFT_REPO_ROOT
for cfg in 4 3 2 1; do
PCFG=$cfg TAG="cfg$cfg split_diag_min=12" python tools/time_step.py 2>&1 | grep RESULT
HDDM_SPLIT_DIAG_MIN=6 PCFG=$cfg TAG="cfg$cfg split_diag_min=6" python tools/time_step.py 2>&1 | grep RESULT
HDDM_SPLIT_DIAG_MIN=48 PCFG=$cfg TAG="cfg$cfg split_diag_min=48" python tools/time_step.py 2>&1 | grep RESULT
done

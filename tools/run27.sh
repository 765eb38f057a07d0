#!/bin/bash
cd $GRAFT_REPO_ROOT
for cfg in 4 3 2 1; do
PCFG=$cfg TAG="cfg$cfg base" python tools/time_step.py 2>&1 | grep RESULT
HDDM_PDL=2 PCFG=$cfg TAG="cfg$cfg pdl2" python tools/time_step.py 2>&1 | grep RESULT
done

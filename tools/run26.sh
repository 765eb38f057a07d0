#!/bin/bash
# session 5: re-measure the launch-structure knobs on the current kernels
cd $GRAFT_REPO_ROOT
for cfg in 4 2 3; do
PCFG=$cfg TAG="cfg$cfg base" python tools/time_step.py 2>&1 | grep RESULT
HDDM_PDL=1 PCFG=$cfg TAG="cfg$cfg pdl" python tools/time_step.py 2>&1 | grep RESULT
HDDM_GROUP_TILES=2 PCFG=$cfg TAG="cfg$cfg group2" python tools/time_step.py 2>&1 | grep RESULT
HDDM_GROUP_TILES=8 PCFG=$cfg TAG="cfg$cfg group8" python tools/time_step.py 2>&1 | grep RESULT
HDDM_GROUP_TILES=8 HDDM_PDL=1 PCFG=$cfg TAG="cfg$cfg group8 pdl" python tools/time_step.py 2>&1 | grep RESULT
done

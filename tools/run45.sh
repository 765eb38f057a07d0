#!/bin/bash
cd $GRAFT_REPO_ROOT
t() { for cfg in 4 2; do env "$@" PCFG=$cfg TAG="cfg$cfg $*" python tools/time_step.py 2>&1 | grep RESULT; done; }
t HDDM_STAGE_CW=32
t HDDM_STAGE_CW=16
t HDDM_STAGE_CW=24
t HDDM_MMA_PULL=0
t HDDM_MMA_BWD=0
t HDDM_MMA_BPULL=1
t HDDM_SUB_RUN=64
t HDDM_SUB_RUN=200
t HDDM_FUSE_BWD=0

#!/bin/bash
cd $GRAFT_REPO_ROOT
for v in 128 129 200; do HDDM_SUB_BWD=$v PCFG=4 TAG="cfg4 SUB_BWD=$v" python tools/time_step.py 2>&1 | grep RESULT; done
for v in 129; do HDDM_SUB_BWD=$v PCFG=2 TAG="cfg2 SUB_BWD=$v" python tools/time_step.py 2>&1 | grep RESULT; done

#!/bin/bash
cd $GRAFT_REPO_ROOT
for cfg in 4 2 3 1; do
PCFG=$cfg TAG="cfg$cfg" python tools/time_step.py 2>&1 | grep RESULT
done
PCFG=4 python tools/solve_once.py 2>&1 | tail -1

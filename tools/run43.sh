#!/bin/bash
# session 5: second pass around the new defaults (FWD_DIV 16, FWD_DIV_SP 8, DIAG_DIV 2, CHECK_CHUNKS 32)
cd $GRAFT_REPO_ROOT
t() { local n=$1 v=$2; shift 2
  for cfg in "$@"; do env $n=$v PCFG=$cfg TAG="cfg$cfg $n=$v" python tools/time_step.py 2>&1 | grep RESULT; done; }
for cfg in 4 3 2 1; do PCFG=$cfg TAG="cfg$cfg newbase" python tools/time_step.py 2>&1 | grep RESULT; done
t HDDM_FWD_DIV 8 4 3 2
t HDDM_FWD_DIV_SP 4 4 3 2
t HDDM_DIAG_DIV 1 4 3 2
t HDDM_CHECK_CHUNKS 16 4 3 2
t HDDM_MMA_DIAG_MIN 16 4 2
t HDDM_SUB_BWD 64 4 2
t HDDM_SUB_BWD 96 4 2

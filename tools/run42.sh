#!/bin/bash
# session 5: runtime knobs re-swept on the final kernels (one at a time around the defaults)
cd $GRAFT_REPO_ROOT
t() { # name value cfgs...
  local n=$1 v=$2; shift 2
  for cfg in "$@"; do env $n=$v PCFG=$cfg TAG="cfg$cfg $n=$v" python tools/time_step.py 2>&1 | grep RESULT; done
}
for cfg in 4 3 2; do PCFG=$cfg TAG="cfg$cfg base" python tools/time_step.py 2>&1 | grep RESULT; done
t HDDM_MMA_FILL 1.15 4 2
t HDDM_MMA_FILL 1.6 4 2
t HDDM_MMA_FILL 2.0 4 2
t HDDM_MMA_DIAG_MIN 16 4 2
t HDDM_MMA_DIAG_MIN 64 4 2
t HDDM_FWD_DIV 16 4 3 2
t HDDM_FWD_DIV 64 4 3 2
t HDDM_FWD_DIV_SP 8 4 3 2
t HDDM_FWD_DIV_SP 32 4 3 2
t HDDM_DIAG_DIV 2 4 3 2
t HDDM_DIAG_DIV 8 4 3 2
t HDDM_FWD_WIDE 8 4 2
t HDDM_FWD_WIDE 32 4 2
t HDDM_FWD_WIDE_SP 3 4 2
t HDDM_FWD_WIDE_SP 12 4 2
t HDDM_SUB_BWD 64 4 2
t HDDM_SUB_BWD 256 4 2
t HDDM_CHECK_CHUNKS 32 4 3 2
t HDDM_CHECK_CHUNKS 128 4 3 2
t HDDM_CTAB_MIN 2 4 2
t HDDM_STAGE_MIN_M 1 4 3
t HDDM_LEAF_STAGE_MIN_M 1 4 3
t HDDM_TILE_MAX 8 4 2
t HDDM_GROUP_TILES 3 4 3 2
t HDDM_GROUP_TILES 6 4 3 2

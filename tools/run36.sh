#!/bin/bash
# session 5: compile-time knob sweep on the box (rebuilds libhddm.so per variant)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() {  # $1 = tag, $2 = EXTRA flags
  make -s -C paper_1807_04180_b200 clean > /dev/null 2>&1
  make -s -j16 -C paper_1807_04180_b200 EXTRA="$2" > /dev/null 2>&1 || { echo "build failed $1"; return; }
  PCFG=4 TAG="$1" python tools/time_step.py 2>&1 | grep RESULT
  PCFG=3 TAG="$1 cfg3" python tools/time_step.py 2>&1 | grep RESULT
}
run base ""
run xfer4 "-DHDDM_XFER_MINB=4"
run xfer2 "-DHDDM_XFER_MINB=2"
run check4 "-DHDDM_CHECK_MINB=4"
run check2 "-DHDDM_CHECK_MINB=2"
run acc2 "-DHDDM_ACC_MINB=2"
run uf2 "-DHDDM_UF=2"
run uf6 "-DHDDM_UF=6"
run ub2 "-DHDDM_UB=2"
run ub6 "-DHDDM_UB=6"
run stage16 "-DHDDM_STAGE_KB=16"
run stage32 "-DHDDM_STAGE_KB=32"
run thr64 "-DHDDM_SOLVE_THREADS=64"
run thr256 "-DHDDM_SOLVE_THREADS=256"
make -s -C paper_1807_04180_b200 clean > /dev/null 2>&1

#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in 4 2 1; do
PCFG=$cfg TAG="cfg$cfg fused fwd" python tools/time_step.py 2>&1 | grep RESULT
HDDM_FUSE_FWD=0 PCFG=$cfg TAG="cfg$cfg nofuse" python tools/time_step.py 2>&1 | grep RESULT
done
PCFG=4 python tools/solve_once.py 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_gpu_ref_live.py -m gpu -q -x > gpurun_out/s5_parity.log 2>&1
echo "pytest rc=$?"; tail -n 3 gpurun_out/s5_parity.log

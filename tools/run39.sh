#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in 4 2 3 1; do
PCFG=$cfg TAG="cfg$cfg" python tools/time_step.py 2>&1 | grep RESULT
HDDM_DEFER_ACC=0 PCFG=$cfg TAG="cfg$cfg nodefer" python tools/time_step.py 2>&1 | grep RESULT
done
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/s5_pytest.log 2>&1
echo "pytest rc=$?"; tail -n 3 gpurun_out/s5_pytest.log

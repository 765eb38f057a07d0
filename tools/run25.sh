#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=cfg4 python tools/stage_prof.py 2>&1 | grep STAGE
PCFG=2 TAG=cfg2 python tools/stage_prof.py 2>&1 | grep STAGE
PCFG=3 TAG=cfg3 python tools/stage_prof.py 2>&1 | grep STAGE
TAG=cfg4 python tools/time_step.py 2>&1 | grep RESULT
PCFG=2 TAG=cfg2 python tools/time_step.py 2>&1 | grep RESULT
PCFG=3 TAG=cfg3 python tools/time_step.py 2>&1 | grep RESULT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref_live.py tests/test_gpu_properties.py tests/test_gpu_shard.py -m gpu -q -x > gpurun_out/s5_parity.log 2>&1
echo "pytest rc=$?"; tail -n 3 gpurun_out/s5_parity.log

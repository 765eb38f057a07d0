#!/bin/bash
# session 5: transfer kernel with members on lanes -- timing, parity, ncu of the stage kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=xfer python tools/stage_prof.py 2>&1 | grep STAGE
PCFG=2 TAG=cfg2 python tools/stage_prof.py 2>&1 | grep STAGE
PCFG=3 TAG=cfg3 python tools/stage_prof.py 2>&1 | grep STAGE
TAG=xfer python tools/time_step.py 2>&1 | grep RESULT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref_live.py tests/test_gpu_properties.py tests/test_gpu_shard.py -m gpu -q -x > gpurun_out/s5_parity.log 2>&1
echo "pytest rc=$?"; tail -n 3 gpurun_out/s5_parity.log
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_rhs_transfer|k_check$|k_accumulate' --launch-skip 12 -c 3 -o gpurun_out/s5_stages -f python tools/stage_prof.py > gpurun_out/s5_stages_ncu.log 2>&1
echo "ncu rc=$?"

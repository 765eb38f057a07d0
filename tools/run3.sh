python -m pytest tests/test_gpu_3d.py -x -q > gpurun_out/t3d.log 2>&1; tail -3 gpurun_out/t3d.log
python tools/cfg5_factor.py 2>&1 | grep RESULT
HDDM3_FACTOR_FMA=1 python tools/cfg5_factor.py 2>&1 | grep RESULT
python tools/cfg5_factor.py 2>&1 | grep RESULT
ncu --set full --clock-control none --import-source on -k regex:k3f_update_mma --launch-skip 300 -c 1 -o gpurun_out/r02_cfg5_update_mma -f python tools/cfg5_factor.py > gpurun_out/ncu_mma.log 2>&1; tail -2 gpurun_out/ncu_mma.log
HDDM3_FACTOR_FMA=1 ncu --set full --clock-control none -k regex:k3f_update --launch-skip 300 -c 1 -o gpurun_out/r02_cfg5_update_fma -f python tools/cfg5_factor.py > gpurun_out/ncu_fma.log 2>&1; tail -2 gpurun_out/ncu_fma.log

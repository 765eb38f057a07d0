ncu --set full --clock-control none --import-source on -k regex:k3s_fpanel --launch-skip 21 -c 1 -o gpurun_out/r02_cfg5_fpanel -f python tools/cfg5_solve_once.py > gpurun_out/ncu_fp.log 2>&1; tail -1 gpurun_out/ncu_fp.log
ncu --set full --clock-control none --import-source on -k regex:k3s_bpanel --launch-skip 16 -c 1 -o gpurun_out/r02_cfg5_bpanel -f python tools/cfg5_solve_once.py > gpurun_out/ncu_bp.log 2>&1; tail -1 gpurun_out/ncu_bp.log
python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r02b.log 2>&1; tail -3 gpurun_out/gputest_r02b.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3

#!/bin/bash
# session-5 baseline: GPU suite, smoke, bench config 4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python bench.py --config 4 > gpurun_out/s5_bench_cfg4.json 2> gpurun_out/s5_bench_cfg4.err
echo "bench rc=$?"
tail -c 600 gpurun_out/s5_bench_cfg4.json
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/s5_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s5_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s5_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/s5_smoke.log
tail -n 3 gpurun_out/s5_pytest.log; tail -n 3 gpurun_out/s5_smoke.log

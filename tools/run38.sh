#!/bin/bash
# session 5 final, part 2: GPU suite, smoke, bench lines of all five configs (default run = config 4)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/final_gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/final_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/final_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/final_smoke.log
tail -n 3 gpurun_out/final_pytest.log; tail -n 3 gpurun_out/final_smoke.log
python bench.py > gpurun_out/final_default.json 2> gpurun_out/final_default.err; echo "default bench rc=$?"
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/final_reference.json 2> gpurun_out/final_reference.err; echo "reference rc=$?"
for c in 1 2 3 4 5; do
  python bench.py --config $c --steps 32 --warmup 3 > gpurun_out/final_cfg$c.json 2> gpurun_out/final_cfg$c.err
  python -c "import json; d=json.load(open('gpurun_out/final_cfg$c.json')); print($c, round(d['value'],1), round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['e2e']['value'], (d['cpu_baseline'] or {}).get('value'), d['clocks'])"
done

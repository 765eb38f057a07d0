for c in 1 2 3 4; do
  python bench.py --config $c --steps 32 --warmup 3 > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err
  python -c "import json; d=json.load(open('gpurun_out/bench_cfg$c.json')); print($c, d['value'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline'])"
done
python tools/fgmres_k.py 2 1 2 4 16 > gpurun_out/fgmres_k_cfg2.jsonl 2>&1; cat gpurun_out/fgmres_k_cfg2.jsonl
HDDM_NO_GRAPHS=1 python tools/fgmres_k.py 2 1 2 4 16 > gpurun_out/fgmres_k_cfg2_nographs.jsonl 2>&1; cat gpurun_out/fgmres_k_cfg2_nographs.jsonl

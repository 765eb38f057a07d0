# round-2 final measurements: bench lines of all five configs, the config-4 launch list
for c in 1 2 3 4 5; do
  python bench.py --config $c --steps 32 --warmup 3 > gpurun_out/final_cfg$c.json 2> gpurun_out/final_cfg$c.err
  python -c "import json; d=json.load(open('gpurun_out/final_cfg$c.json')); print($c, round(d['value'],1), round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['e2e']['value'], (d['cpu_baseline'] or {}).get('value'), d['clocks'])"
done
for c in 4 2; do
HDDM_NO_GRAPHS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base --csv --log-file gpurun_out/final_launches_cfg$c.csv python bench.py --config $c --steps 3 --warmup 1 --skip-e2e --skip-cpu > gpurun_out/final_ncu$c.log 2>&1
python tools/ncu_step.py gpurun_out/final_launches_cfg$c.csv gpurun_out/final_step_summary_cfg$c.json | tail -3
done

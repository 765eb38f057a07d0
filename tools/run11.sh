for c in 4 2; do for o in asc desc; do
HDDM_GROUP_ORDER=$o python bench.py --config $c --steps 32 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/ord_${c}_${o}.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ord_${c}_${o}.json')); print('cfg', $c, '$o', 'ms/step', round(d['ms_per_step'],4), 'solve ms', round(d['roofline']['ms_per_launch'],4))"
done; done

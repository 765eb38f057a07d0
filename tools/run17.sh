for c in 4 2; do for f in 0 1.15 1.3 1.6 9; do
HDDM_MMA_FILL=$f python bench.py --config $c --steps 32 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/fill_${c}_${f}.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/fill_${c}_${f}.json')); print('cfg', $c, 'fill', $f, 'ms/step', round(d['ms_per_step'],4), 'solve ms', round(d['roofline']['ms_per_launch'],4))"
done; done

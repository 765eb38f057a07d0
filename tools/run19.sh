for c in 4 2; do for dm in 16 32 64 100000; do
HDDM_MMA_DIAG_MIN=$dm python bench.py --config $c --steps 32 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/dm_${c}_${dm}.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/dm_${c}_${dm}.json')); print('cfg', $c, 'diag_min', $dm, 'ms/step', round(d['ms_per_step'],4), 'solve ms', round(d['roofline']['ms_per_launch'],4))"
done; done

for c in 4 2; do for v in 0 1; do
HDDM_MMA_BWD=$v python bench.py --config $c --steps 32 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/mmab_${c}_${v}.json 2>gpurun_out/mmab_${c}_${v}.err
python -c "import json; d=json.load(open('gpurun_out/mmab_${c}_${v}.json')); print('cfg', $c, 'mma_bwd', $v, 'ms/step', round(d['ms_per_step'],4), 'solve ms', round(d['roofline']['ms_per_launch'],4), d['refine'])" || tail -3 gpurun_out/mmab_${c}_${v}.err
done; done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py -x -q 2>&1 | tail -2

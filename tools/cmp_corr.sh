set -x
for cfg in 3 4; do
for cap in 4 1073741824; do
HDDM_CORR_GROUP_TILES=$cap python bench.py --config $cfg --steps 16 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/corr_${cfg}_${cap}.json 2>gpurun_out/corr_${cfg}_${cap}.err
python -c "
import json; d=json.load(open('gpurun_out/corr_${cfg}_${cap}.json'))
print('cfg',$cfg,'cap',$cap,'ms/step',round(d['ms_per_step'],4),'solve ms',round(d['roofline']['ms_per_launch'],4),'refine',d['refine'])"
done; done

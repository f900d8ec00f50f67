# A/B of the one-CTA sort cutoff (VR_SMALL_SORT_MAX): 8192 = the old behaviour (rs_small up
# to RS_SMALL_CAP), 2048 = the default (clusters of 2-4 CTAs above it).  GPU box via gpurun.
for m in 8192 2048 8192 2048; do
  VR_SMALL_SORT_MAX=$m timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-target > gpurun_out/abs_$m.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/abs_$m.json')); print('M=$m', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages_ms'].items()})" >> gpurun_out/abs.txt
done
cat gpurun_out/abs.txt

# Sweep of the small-sort cutoff (VR_SMALL_SORT_MAX) and the cluster tile (VR_CL_TILE) on c2.
for cfg in "2048 2048" "512 2048" "1024 2048" "2048 1024" "512 1024" "2048 512" "2048 2048"; do
  set -- $cfg
  VR_SMALL_SORT_MAX=$1 VR_CL_TILE=$2 timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-target > gpurun_out/abss.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/abss.json')); print('SMALL=$1 TILE=$2', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages_ms'].items()})" >> gpurun_out/abss.txt
done
cat gpurun_out/abss.txt

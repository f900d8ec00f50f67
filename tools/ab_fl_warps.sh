# A/B of the flat-enumeration chunk sizing target (warps per SM; affects dimensions whose
# C(n, D+1) gives chunks below 1024, e.g. c2 dimension 2).  Run on the GPU box via gpurun.
python paper_2502_05063_b200/build.py > /dev/null 2>&1 || exit 1
for w in ${VR_AB_WARPS:-24 32 48 64 96 24}; do
  VR_FL_WARPS=$w timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-target > gpurun_out/abw_$w.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/abw_$w.json')); print('W=$w', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages_ms'].items()})" >> gpurun_out/abw.txt
done
cat gpurun_out/abw.txt

# A/B of k_enumerate_flat min-blocks-per-SM (run on the GPU box via gpurun; rebuilds libvr per variant)
set -x
for mb in 4 5 6; do
  sed -i "s/__launch_bounds__(HP_THREADS, [0-9]) k_enumerate_flat/__launch_bounds__(HP_THREADS, $mb) k_enumerate_flat/" paper_2502_05063_b200/csrc/hotpath.cu
  python paper_2502_05063_b200/build.py > gpurun_out/ab_build_$mb.log 2>&1 || continue
  for rep in 1 2; do
  timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-target > gpurun_out/ab_${mb}_${rep}.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab_${mb}_${rep}.json')); print('MB=$mb', d['ms_per_step'], d['stages_ms'])" >> gpurun_out/ab.txt
  done
done
cat gpurun_out/ab.txt
sed -i "s/__launch_bounds__(HP_THREADS, [0-9]) k_enumerate_flat/__launch_bounds__(HP_THREADS, 4) k_enumerate_flat/" paper_2502_05063_b200/csrc/hotpath.cu

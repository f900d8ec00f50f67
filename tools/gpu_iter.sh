python paper_2502_05063_b200/build.py >/dev/null && python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-target > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); print(d['ms_per_step'], d['stages_ms'], d['roofline']['frac'], d['wall_s'])"

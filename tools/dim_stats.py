"""Per-dimension device times and counters of one public call (diagnostics):
python tools/dim_stats.py c5_o3_4096 3 [repeats]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_05063_b200 as vr  # noqa: E402
from datagen import clouds as G  # noqa: E402

cfg = G.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5_o3_4096"]
D = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.max_dim
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
lt = cfg.lower_tri()
for _ in range(reps):
    t0 = time.perf_counter()
    bc = vr.barcodes(lt, cfg.n, D, cfg.threshold)
    wall = time.perf_counter() - t0
    print(f"wall {wall:.3f} s")
    for d in range(D + 1):
        s = bc.stats[d]
        print(d, {k: (round(v, 3) if isinstance(v, float) else v) for k, v in s.items()})

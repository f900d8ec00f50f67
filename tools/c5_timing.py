"""Time the north-star workload (config 5 at max_dim 2) end to end, with stats (diagnostics)."""
import os, sys, time
root = sys.argv[1] if len(sys.argv) > 1 else os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
import paper_2502_05063_b200 as vr
from datagen import clouds as G
print(vr.__file__)
c5 = G.CONFIGS["c5_o3_4096"]
lt = c5.lower_tri()
for i in range(4):
    t0 = time.perf_counter()
    b = vr.barcodes(lt, c5.n, 2, c5.threshold)
    dt = time.perf_counter() - t0
    print(round(dt, 3), [(d, {k: round(v, 1) for k, v in b.stats[d].items() if k.startswith("ms_")}) for d in range(3)], flush=True)

"""Time vr_min_cost_flow on a dumped network (tools/dump_w1_net.py); host only."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2502_05063_b200 as vr
z = dict(np.load(sys.argv[1]))
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    t0 = time.perf_counter()
    v, st = vr.min_cost_flow(z["supply"], z["tail"], z["head"], z["cost"])
    print(round(time.perf_counter() - t0, 3), v, st, flush=True)

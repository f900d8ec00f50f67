"""Sweep the phase-1 scan budget (vr_options.apparent_steps) on a config: device ms per stage
of the hot path (plan replay, median of 10).  Diagnostics: python tools/steps_sweep.py c5_o3_4096 3 16 32 64 128"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_05063_b200 as vr  # noqa: E402
from datagen import clouds as G  # noqa: E402

cfg = G.CONFIGS[sys.argv[1]]
D = int(sys.argv[2])
lt = torch.from_numpy(cfg.lower_tri()).cuda()
for s in [int(x) for x in sys.argv[3:]]:
    plan = vr.Plan(lt, cfg.n, D, cfg.threshold, apparent_steps=s)
    rows = []
    for _ in range(10):
        plan.replay()
        rows.append(plan.timing())
    med = {k: round(statistics.median(r[k] for r in rows), 3) for k in ("ms_tables", "ms_enumerate", "ms_resolve", "ms_sort")}
    st = plan.result.stats
    print(s, med, round(sum(med.values()), 3), "queued", [st[d]["queued"] for d in range(1, D + 1)], flush=True)
    plan.close()

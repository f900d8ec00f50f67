"""Hot-path device time vs the phase-1 tuning knobs (diagnostics)."""
import itertools, json, math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2502_05063_b200 as vr
from datagen import clouds as G

names = [a for a in sys.argv[1:] if not a.startswith("--")]
combos = [(32, 2), (4, 3), (8, 3), (12, 3), (16, 3), (24, 3), (32, 3)]
for name in names:
    cfg = G.CONFIGS[name]
    lt = torch.from_numpy(cfg.lower_tri()).cuda()
    ref = None
    for steps, var in combos:
        plan = vr.Plan(lt, cfg.n, cfg.max_dim, cfg.threshold, apparent_steps=steps, scan_variant=var)
        bars = [p.tobytes() for p in plan.result.pairs]
        if ref is None:
            ref = bars
        assert bars == ref, "tuning changed the barcode"
        for _ in range(3):
            plan.replay()
        acc = {"ms_tables": 0, "ms_enumerate": 0, "ms_resolve": 0, "ms_sort": 0}
        for _ in range(5):
            plan.replay()
            t = plan.timing()
            for k in acc:
                acc[k] += t[k] / 5
        q = sum(plan.result.stats[d]["queued"] for d in range(1, cfg.max_dim + 1))
        print(json.dumps({"config": name, "steps": steps, "variant": var, "queued": q,
                          **{k: round(v, 3) for k, v in acc.items()}, "total": round(sum(acc.values()), 3)}), flush=True)
        plan.close()

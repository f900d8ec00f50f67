"""Hot-path device time vs the phase-1 tuning knobs (diagnostics)."""
import itertools, json, math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2502_05063_b200 as vr
from datagen import clouds as G

names = [a for a in sys.argv[1:] if not a.startswith("--")]
steps_list = [32]
grabs = [1, 2, 4, 8]
variants = [1, 2]
for name in names:
    cfg = G.CONFIGS[name]
    lt = torch.from_numpy(cfg.lower_tri()).cuda()
    for steps, grab, var in itertools.product(steps_list, grabs, variants):
        plan = vr.Plan(lt, cfg.n, cfg.max_dim, cfg.threshold, apparent_steps=steps, rows_per_grab=grab, scan_variant=var)
        for _ in range(3):
            plan.replay()
        acc = {"ms_tables": 0, "ms_enumerate": 0, "ms_resolve": 0, "ms_sort": 0}
        for _ in range(5):
            plan.replay()
            t = plan.timing()
            for k in acc:
                acc[k] += t[k] / 5
        q = sum(plan.result.stats[d]["queued"] for d in range(1, cfg.max_dim + 1))
        print(json.dumps({"config": name, "steps": steps, "grab": grab, "variant": var, "queued": q,
                          **{k: round(v, 3) for k, v in acc.items()}, "total": round(sum(acc.values()), 3)}), flush=True)
        plan.close()

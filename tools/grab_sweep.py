"""Hot-path device time vs rows_per_grab (diagnostics)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_05063_b200 as vr
from datagen import clouds as G
for name in sys.argv[1:]:
    cfg = G.CONFIGS[name]
    lt = torch.from_numpy(cfg.lower_tri()).cuda()
    for grab in [int(g) for g in os.environ.get("GRABS", "1,2,4,8,16,32,64").split(",")]:
        plan = vr.Plan(lt, cfg.n, cfg.max_dim, cfg.threshold, rows_per_grab=grab)
        for _ in range(3):
            plan.replay()
        acc = {"ms_tables": 0, "ms_enumerate": 0, "ms_resolve": 0, "ms_sort": 0}
        for _ in range(5):
            plan.replay()
            t = plan.timing()
            for k in acc:
                acc[k] += t[k] / 5
        print(json.dumps({"config": name, "grab": grab, **{k: round(v, 4) for k, v in acc.items()}}), flush=True)
        plan.close()

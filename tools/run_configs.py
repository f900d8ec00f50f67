"""Run vr_barcodes on the BASELINE configs and print per-dimension stats (diagnostics)."""
from __future__ import annotations

import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2502_05063_b200 as vr  # noqa: E402
from datagen import clouds as G  # noqa: E402


def main(names, max_dim=None):
    for name in names:
        cfg = G.CONFIGS[name]
        D = cfg.max_dim if max_dim is None else max_dim
        t0 = time.perf_counter()
        lt = cfg.lower_tri()
        tg = time.perf_counter() - t0
        vr.barcodes(lt, cfg.n, D, cfg.threshold)  # warm
        t0 = time.perf_counter()
        bc = vr.barcodes(lt, cfg.n, D, cfg.threshold)
        wall = time.perf_counter() - t0
        out = {"config": name, "D": D, "gen_s": round(tg, 2), "wall_s": round(wall, 4), "t": bc.threshold,
               "bars": [len(p) for p in bc.pairs]}
        for d in range(D + 1):
            s = bc.stats[d]
            out[f"d{d}"] = {k: (round(v, 3) if isinstance(v, float) else v) for k, v in s.items()}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    md = None
    for a in sys.argv[1:]:
        if a.startswith("--max-dim="):
            md = int(a.split("=")[1])
    main(args or ["c1_circle64", "c2_s3_192", "c4a_sierpinski512", "c3_trefoil1000"], md)

"""One config's full barcodes from the library against the oracle-pinned single-threaded
cpu_ripser (diagnostics / evidence; the GPU tests do this for c2, c3 and c5):
python tools/full_bars_vs_cpu_ripser.py c4b_torus2000"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cpu_ripser as RS  # noqa: E402
import paper_2502_05063_b200 as vr  # noqa: E402
from datagen import clouds as G  # noqa: E402


def sorted_bars(p):
    p = np.asarray(p, np.float32).reshape(-1, 2)
    return p[np.lexsort((p[:, 1], p[:, 0]))]


cfg = G.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4b_torus2000"]
lt = cfg.lower_tri()
t0 = time.perf_counter()
bc = vr.barcodes(lt, cfg.n, cfg.max_dim, cfg.threshold)
t_gpu = time.perf_counter() - t0
t0 = time.perf_counter()
pairs, st = RS.barcode(lt, cfg.n, cfg.max_dim, bc.threshold)
t_cpu = time.perf_counter() - t0
eq = [bool(np.array_equal(sorted_bars(pairs[d]).view(np.uint32), sorted_bars(bc.pairs[d]).view(np.uint32)))
      for d in range(cfg.max_dim + 1)]
print(json.dumps({"config": cfg.name, "max_dim": cfg.max_dim, "bars_equal_per_dim": eq,
                  "bars": [len(bc.pairs[d]) for d in range(cfg.max_dim + 1)],
                  "library_wall_s": round(t_gpu, 2), "cpu_ripser_wall_s": round(t_cpu, 2)}))

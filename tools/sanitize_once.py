"""One public call per config for compute-sanitizer runs (small configs):
python tools/sanitize_once.py c1_circle64 c4a_sierpinski512 [--sparse] [--ranks 2]"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2502_05063_b200 as vr  # noqa: E402
from datagen import clouds as G  # noqa: E402

names = [a for a in sys.argv[1:] if not a.startswith("--")]
for name in names:
    cfg = G.CONFIGS[name]
    lt = cfg.lower_tri()
    a = vr.barcodes(lt, cfg.n, cfg.max_dim, cfg.threshold)
    b = vr.barcodes(lt, cfg.n, cfg.max_dim, cfg.threshold, sparse_mode=2)  # the output-sensitive kernels too
    same = all(np.array_equal(a.pairs[d], b.pairs[d]) for d in range(cfg.max_dim + 1))
    print(name, [len(p) for p in a.pairs], "dense == sparse:", same, flush=True)
c5 = G.CONFIGS["c5_o3_4096"]
p = c5.patch(300)
r = vr.barcodes(p, 300, 3, 1.4)
print("c5 patch 300", [len(x) for x in r.pairs], flush=True)

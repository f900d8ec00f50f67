"""One public call on a named config (for ncu captures): python tools/profile_once.py c2_s3_192 3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_05063_b200 as vr  # noqa: E402
from datagen import clouds as G  # noqa: E402

cfg = G.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2_s3_192"]
D = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.max_dim
bc = vr.barcodes(cfg.lower_tri(), cfg.n, D, cfg.threshold)
print([len(p) for p in bc.pairs])

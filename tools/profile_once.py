"""One public call on a named config (for ncu captures):
python tools/profile_once.py c2_s3_192 3 [--hot]   (--hot: hot path only, no host residual)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_05063_b200 as vr  # noqa: E402
from datagen import clouds as G  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
cfg = G.CONFIGS[args[0] if args else "c2_s3_192"]
D = int(args[1]) if len(args) > 1 else cfg.max_dim
bc = vr.barcodes(cfg.lower_tri(), cfg.n, D, cfg.threshold, hot_path_only="--hot" in sys.argv)
print([len(p) for p in bc.pairs], [bc.stats[d]["ms_enumerate"] for d in range(D + 1)])

"""Dump the PDoptFlow network of a synthetic pair (diagnostics for netsimplex work)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2502_05063_b200 as vr
from datagen import diagrams as PD
n = int(sys.argv[1]); s = float(sys.argv[2]); out = sys.argv[3]
A, B = PD.gaussian(n, 1), PD.gaussian(n, 2)
net = vr.w1_network(A, B, s=s, seed=0)
np.savez_compressed(out, supply=net["supply"], tail=net["tail"], head=net["head"], cost=net["cost"])
v, st = vr.w1(A, B, s=s, seed=0)
print(n, s, v, {k: st[k] for k in ("nodes", "arcs", "pivots", "degenerate", "blocks", "ms_simplex", "ms_pricing", "ms_update")})

#!/usr/bin/env python
"""PAPER.md §5.6.6 at scale: the apparent-pair fraction of dimension 1 for
random distance matrices (SURVEY.md §8(f) NEXT-2's scale smoke test).

Input: a uniformly random permutation of 1..n(n-1)/2 fills the lower triangle
(Obs 5.6.8: only the order matters; the permutation index k is mapped to the fp32 value
with bit pattern 0x3F800000 + k — distinct, positive, order-preserving).  Only the GPU hot
path of dimension 1 runs (vr_options.hot_path_only: enumeration, apparent test, compaction,
sort — no residual reduction).  Reported: apparent pairs / C(n, 2) (the paper's "apparent
fraction" of the 1-dimensional coboundary matrix), apparent / survivors (edges <= R), the
Theorem 5.4.2 bound (n-2)/n, and the paper's printed values at n = 10000 and 20000
(0.991127743, 0.993733522, averages over its samples).
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

PAPER = {10000: 0.991127743, 20000: 0.993733522}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="*", default=[1000, 2000, 5000, 10000, 20000])
    ap.add_argument("--samples", type=int, default=3)
    args = ap.parse_args()
    import paper_2502_05063_b200 as vr
    for n in args.n:
        N = n * (n - 1) // 2
        fr, fs, ts = [], [], []
        for s in range(args.samples):
            rng = np.random.default_rng(1000 + s)
            perm = rng.permutation(N).astype(np.uint32)
            vals = (perm + np.uint32(0x3F800000)).view(np.float32)
            lt = torch.from_numpy(vals).cuda()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            bc = vr.barcodes_device(lt, n, 1, math.inf, hot_path_only=True)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
            surv, app = bc.stats[1]["survivors"], bc.stats[1]["apparent"]
            fr.append(app / N)
            fs.append(app / max(surv, 1))
            del lt
        line = {"n": n, "samples": args.samples, "apparent_fraction": float(np.mean(fr)),
                "apparent_fraction_std": float(np.std(fr)), "apparent_over_survivors": float(np.mean(fs)),
                "bound_thm_5_4_2": (n - 2) / n, "paper": PAPER.get(n), "s_per_sample": float(np.mean(ts))}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

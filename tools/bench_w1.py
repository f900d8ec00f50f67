#!/usr/bin/env python
"""PDoptFlow row measurement: one JSON line per workload.

Workloads (datagen/diagrams.py, seeded): pairs of Gaussian diagrams as in Fig 6.1
 of n points each, and a pair of clustered (2^8-level) diagrams.
  value        points/s = (|A| + |B|) / wall time of vr_w1 (host arrays in, W1 out)
  stages       device/host stage times from vr_w1_stats
  roofline     the dominant GPU kernel, k_rwmd: fp64 FMA-bound brute-force nearest
               neighbours, 3 fp64 ops (2 sub + 1 fma ... counted as 4 flops) per pair
  cpu_baseline the oracle (exact W1 by assignment, one core) on the first `sample` points
               of each diagram, scaled to points/s
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from datagen import diagrams as PD  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="*", default=[10000, 20000, 50000])
    ap.add_argument("--s", type=float, nargs="*", default=[18.0])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--sample", type=int, default=1200)
    ap.add_argument("--no-oracle", action="store_true")
    args = ap.parse_args()
    import paper_2502_05063_b200 as vr
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    work = []
    for n in args.n:
        work.append((f"gaussian_{n}", PD.gaussian(n, 1), PD.gaussian(n, 2)))
    work.append(("clustered_50000", PD.clustered(50000, 3), PD.clustered(50000, 4)))
    # the diagrams the library produces: all finite bars of config 3
    # (trefoil tube, n = 1000, dims 0-2) against those of a re-sampled copy (seed + 100)
    from datagen import clouds as G
    c3 = G.CONFIGS["c3_trefoil1000"]
    vd = []
    for seed_shift in (0, 100):
        cfg = c3 if seed_shift == 0 else G.Config(**{**c3.__dict__, "seed": c3.seed + seed_shift})
        bc = vr.barcodes(cfg.lower_tri(), cfg.n, 2, cfg.threshold)
        P = np.concatenate([p for p in bc.pairs])
        vd.append(P[np.isfinite(P[:, 1])].astype(np.float32))
    work.append(("vr_c3_bars_vs_resampled", vd[0], vd[1]))
    for name, A, B in work:
        for s in args.s:
            vr.w1(A[:100], B[:100], s=s)  # warm
            walls, vals, st = [], [], None
            for _ in range(args.steps):
                t0 = time.perf_counter()
                v, st = vr.w1(A, B, s=s, seed=0)
                walls.append(time.perf_counter() - t0)
                vals.append(v)
            wall = statistics.median(walls)
            pairs = len(A) * len(B) * 2
            # fp64 peak derived from unit counts and clock: 148 SMs x 64 FP64 FMA lanes x 2
            # flops x sm_max_mhz; the kernel's algorithmic flops = 4 per (u, v) pair (2 sub,
            # 1 mul, 1 fma) in both directions
            fp64_peak = 148 * 64 * 2 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
            rw_ms = st["ms_rwmd"]
            achieved = 4 * pairs / (rw_ms / 1e3) / 1e12 if rw_ms > 0 else None
            line = {"metric": "PDoptFlow W1 points/s", "value": (len(A) + len(B)) / wall, "unit": "points/s",
                    "higher_is_better": True, "steps": args.steps, "dtype": "f64", "data": "synthetic",
                    "config": {"workload": name, "s": s, "points_a": len(A), "points_b": len(B)},
                    "wall_s": wall, "w1": vals[0], "deterministic": len(set(vals)) == 1,
                    "stats": st,
                    "roofline": {"bound": "fp64", "kernel": "k_rwmd", "achieved": achieved, "peak": fp64_peak,
                                 "unit": "TFLOP/s", "frac": achieved / fp64_peak if achieved else None, "traffic": None,
                                 "peak_source": "derived: 148 SM x 64 FP64 lanes x 2 x sm_max_mhz"}}
            if not args.no_oracle:
                from oracle import w1 as W
                k = args.sample
                t0 = time.perf_counter()
                W.w1_exact(A[:k], B[:k])
                dt = time.perf_counter() - t0
                line["cpu_baseline"] = {"value": 2 * k / dt, "unit": "points/s", "cores": 1, "kind": "oracle",
                                        "sample": f"first {k} points of each diagram, exact W1 by assignment", "wall_s": dt}
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""HYPHA row measurement: one JSON line per matrix.

Matrices (synthetic, tests/_boundary.py), the two Table 4.1 rows we can rebuild without
datasets: the 18-sphere (every proper face of the 19-simplex, 2^20 - 2 columns, ordered by
dimension then colex) and a mumford-shaped matrix (the 4-skeleton of the Rips filtration
of 50 random points, 2.37e6 columns, ordered by diameter, dimension, colex).

  value       columns / s of vr_hypha_pivots end to end (host CSC in, low[] out: H2D,
              the three GPU-scan kernels, D2H, host compression + reduction), median of K
  gpu_scan    the scan alone (CUDA events around the memsets + three kernels), and its
              stable-column throughput — the quantity of Fig 4.9
  roofline    HBM: algorithmic bytes of the scan / scan time
  cpu_baseline the oracle's Alg 2 (oracle.reduce_csc, one core) on the same matrix
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import _boundary as B  # noqa: E402
from datagen import clouds as G  # noqa: E402


def scan_bytes(ptr, nnz, unstable):
    n = ptr.size - 1
    # memsets (left, lookup 4 B, stable 1 B) + k_set_leftmost (col_ptr, rows, left written
    # once, low written) + k_set_lookup (low, left gather, lookup write, stable write)
    # + k_set_unstable (stable read, u write)
    return 9 * n + (8 * n + 4 * nnz + 4 * n + 4 * n) + (4 * n + 4 * n + 4 * n + 1 * n) + (1 * n + 4 * unstable)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--matrix", default="all", choices=["all", "sphere18", "mumford50"])
    ap.add_argument("--no-oracle", action="store_true")
    args = ap.parse_args()
    import paper_2502_05063_b200 as vr
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    mats = {}
    if args.matrix in ("all", "sphere18"):
        mats["sphere18"] = B.sphere_fast(19)
    if args.matrix in ("all", "mumford50"):
        mats["mumford50_4skel"] = B.rips_fast(G.random_cloud(50, 1), 50, 3)
    for name, (ptr, rows, dims) in mats.items():
        vr.hypha_pivots(ptr, rows, dims)  # warm (context, module load)
        walls, scans, st = [], [], None
        for _ in range(args.steps):
            t0 = time.perf_counter()
            low, st = vr.hypha_pivots(ptr, rows, dims)
            walls.append(time.perf_counter() - t0)
            scans.append(st["ms_gpu_scan"])
        ncols = ptr.size - 1
        wall = statistics.median(walls)
        scan_ms = statistics.median(scans)
        byts = scan_bytes(ptr, int(ptr[-1]), st["unstable"])
        achieved = byts / (scan_ms / 1e3) / 1e9
        line = {
            "metric": "HYPHA boundary-matrix pivots, columns/s", "value": ncols / wall, "unit": "columns/s",
            "higher_is_better": True, "steps": args.steps, "dtype": "int32", "data": "synthetic",
            "config": {"workload": name, "columns": ncols, "nnz": int(ptr[-1]), "twist": True, "compression": True},
            "wall_s": wall,
            "gpu_scan": {"ms": scan_ms, "stable": st["stable"], "stable_per_s": st["stable"] / (scan_ms / 1e3)},
            "host_ms": st["ms_host"], "stats": st,
            "roofline": {"bound": "hbm", "kernel": "GPU-scan (k_set_leftmost+k_set_lookup+k_set_unstable)",
                         "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / peaks["hbm_gbs"], "traffic": None, "bytes": byts},
        }
        if not args.no_oracle:
            from oracle import oracle as O
            t0 = time.perf_counter()
            ref = O.reduce_csc(ptr, rows)
            dt = time.perf_counter() - t0
            assert np.array_equal(ref, low), name
            line["cpu_baseline"] = {"value": ncols / dt, "unit": "columns/s", "cores": 1, "kind": "oracle",
                                    "sample": f"the whole {name} matrix, Alg 2 left to right", "wall_s": dt}
            line["parity"] = "low[] identical to the oracle"
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

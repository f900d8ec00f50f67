#!/usr/bin/env python
"""bench.py — hot-path simplices/s of the B200 Vietoris–Rips barcode path (one JSON line).

Metric (BASELINE.json `metric`): "VR barcode wall-time (s) and hot-path simplices/sec".
  value   = hot-path simplices/s: sum over d = 1..max_dim of the d-simplices with
            diam <= t (the survivors, a method-independent count) divided
            by the device time of one pass of the whole GPU hot path (a0 tables, a1
            enumeration + threshold, a5 apparent test, a2 clearing, a3/a6 compaction, a4
            radix sort) — vr_plan_replay, inputs resident in HBM, CUDA events on the
            launching stream, L2 flushed (256 MiB write) before every timed step.
  e2e     = the same numerator over the wall time of the public host-pointer call
            vr_barcodes (H2D of the fp32 lower triangle, dimension 0, every dimension's
            hot path, the host residual reduction, D2H of the barcode) — also reported as
            seconds per barcode ("wall_s").
Default workload: BASELINE.json configs[4], the config the metric is quoted on: n = 4096
points of an O(3)-shaped cloud, max_dim 3, threshold 1.4 (output-sensitive mode).  The
north-star target (the same input at max_dim 2 under 1 s end to end) and the other configs
(c2, c3, c4a, c4b: hot path and end to end) are extra keys of the same line.

Roofline: the integer-ALU and L2 peaks are MEASURED on the box (vr_probe_peaks) and are the
denominators of the dominant kernel's fraction.

Multi-GPU: `--gpus N` without torchrun re-launches itself under torch.distributed.run with N
ranks (one process per GPU); under torchrun the workload is sharded over the ranks inside
libvr (NCCL communicator from a unique id shared by torch.distributed; strong scaling) and
value = survivors / max-over-ranks step time.  --impl reference times the CPU
oracle (explicit boundary matrix + Alg 2) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from datagen import clouds as G  # noqa: E402

METRIC = "hot-path simplices/s (VR barcodes, dims 1..max_dim)"
# the JSON line goes to the process's real stdout; everything else a library may print on
# fd 1 (e.g. NCCL's version banner at communicator init) is sent to stderr (see main())
OUT = sys.stdout
UNIT = "simplices/s"
HEADLINE = "c5_o3_4096"
EXTRA_CONFIGS = ["c2_s3_192", "c3_trefoil1000", "c4a_sierpinski512", "c4b_torus2000"]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=HEADLINE, choices=sorted(G.CONFIGS))
    ap.add_argument("--max-dim", type=int, default=None)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ripser", action="store_true", help="skip the single-threaded Ripser-style CPU run")
    ap.add_argument("--no-extra", action="store_true", help="skip the other configs' lines")
    ap.add_argument("--sample", type=int, default=None, help="oracle sample size (points)")
    ap.add_argument("--no-target", action="store_true", help="skip the north-star target run (config 5, max_dim 2)")
    ap.add_argument("--sharded", action="store_true", help="use the sharded (multi-GPU) path even at N=1")
    return ap.parse_args()


def workload(args):
    cfg = G.CONFIGS[args.config]
    D = cfg.max_dim if args.max_dim is None else args.max_dim
    return cfg, D


def config_obj(cfg, D, extra=None):
    o = {"workload": f"{cfg.name}: n={cfg.n} {cfg.shape} cloud, max_dim={D}, "
                     f"threshold={'R (enclosing radius)' if math.isinf(cfg.threshold) else cfg.threshold}",
         "n": cfg.n, "max_dim": D, "threshold": None if math.isinf(cfg.threshold) else cfg.threshold,
         "seed": cfg.seed, "l2": "flushed before every timed step (256 MiB write)"}
    if extra:
        o.update(extra)
    return o


# ------------------------------------------------------------------ clocks during the timed region
class ClockSampler:
    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index, self.samples, self._stop = index, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                self.samples.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return None
        sm = [int(s[0]) for s in self.samples if s and s[0].isdigit()]
        mx = [int(s[1]) for s in self.samples if len(s) > 1 and s[1].isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples if len(s) >= 7 for i in range(4) if s[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------ CPU baselines (pinned to one core)
def host_info():
    return {"nproc": os.cpu_count(), "cpu": _cpu_model()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


class OneCore:
    """Pins the calling thread to one CPU for the duration (the single-threaded baselines)."""

    def __enter__(self):
        self.prev = os.sched_getaffinity(0)
        self.cpu = min(self.prev)
        os.sched_setaffinity(0, {self.cpu})
        return self

    def __exit__(self, *a):
        os.sched_setaffinity(0, self.prev)


def oracle_sample(cfg, D, m):
    """The oracle on a bounded sample of the workload: the first m points for the full-Rips
    configs; for a thresholded config (config 5) the m points nearest to point 0 (a patch at
    the cloud's own density — a first-m subsample is nearly empty at t = 1.4)."""
    from oracle import oracle as O
    thresholded = not math.isinf(cfg.threshold)
    lt = cfg.patch(m) if thresholded else cfg.lower_tri(m)
    t = cfg.threshold if thresholded else O.enclosing_radius(lt, m)
    t0 = time.perf_counter()
    b = O.barcode(lt, m, D, t)
    dt = time.perf_counter() - t0
    return sum(b.n_simplices[1:D + 1]), dt, ("patch of the %d points nearest to point 0" % m if thresholded
                                             else "first %d points" % m)


def default_sample(cfg, D):
    if not math.isinf(cfg.threshold):
        return 118  # the oracle's dense position index caps C(m, D+2) at 2e8
    return {1: 64, 2: 64, 3: 56}.get(D, 40) if cfg.n > 64 else cfg.n


def cpu_baseline(cfg, D, m):
    with OneCore() as c:
        surv, dt, what = oracle_sample(cfg, D, m)
    hi = host_info()
    return {"value": surv / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{what} of {cfg.name} (same generator), max_dim={D}, same threshold rule: "
                      f"{surv} simplices in dims 1..{D}, {dt:.2f} s single-threaded (explicit boundary "
                      f"matrix + standard reduction, no clearing/cohomology/apparent pairs); 1 of {hi['nproc']} "
                      f"cores ({hi['cpu']}), pinned to CPU {c.cpu}"}


def ripser_style_run(cfg, D, threshold, gpu_pairs):
    """BASELINE.json north_star: "a single-threaded Ripser-style CPU run timed on the box's
    own host cores in the same run" — cpu_ripser/ (implicit cohomology, clearing, emergent
    pairs, heap columns, neighbour lists for sparse thresholds; §5.2) on the FULL
    workload at the threshold the GPU path used, its bars compared with the GPU path's."""
    import cpu_ripser as RS
    RS.build()
    lt = cfg.lower_tri()
    with OneCore() as c:
        t0 = time.perf_counter()
        pairs, st = RS.barcode(lt, cfg.n, D, threshold)
        dt = time.perf_counter() - t0
    surv = sum(st[d]["simplices"] for d in range(1, D + 1))

    def srt(a):
        a = np.asarray(a, np.float32).reshape(-1, 2)
        return a[np.lexsort((a[:, 1], a[:, 0]))] if len(a) else a
    same = all(np.array_equal(srt(pairs[d]), srt(gpu_pairs[d])) for d in range(D + 1))
    hi = host_info()
    return {"value": surv / dt, "unit": UNIT, "cores": 1, "kind": "ripser-style", "wall_s": dt,
            "bars_equal_gpu": bool(same),
            "per_dim_ms": [round(s["ms"], 1) for s in st],
            "sample": f"full {cfg.name} workload, max_dim={D}, t={threshold:.6g}: {surv} simplices in dims 1..{D}, "
                      f"single-threaded cpu_ripser (implicit coboundary cohomology + clearing + emergent pairs); "
                      f"1 of {hi['nproc']} cores ({hi['cpu']}), pinned to CPU {c.cpu}"}


# ------------------------------------------------------------------ arms
def run_reference(args, rank, world):
    cfg, D = workload(args)
    if rank != 0:
        return
    m = min(args.sample or default_sample(cfg, D), cfg.n)
    from oracle import oracle as O
    O.build()
    with OneCore() as c:
        for _ in range(args.warmup):
            oracle_sample(cfg, D, m)
        tot_s, tot_t = 0, 0.0
        for _ in range(args.steps):
            s, dt, what = oracle_sample(cfg, D, m)
            tot_s += s
            tot_t += dt
    v = tot_s / tot_t
    hi = host_info()
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * tot_t / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_obj(cfg, D, {"sample_points": m}),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{what} of {cfg.name} per step, max_dim={D}; 1 of {hi['nproc']} cores, "
                                       f"pinned to CPU {c.cpu}"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), file=OUT, flush=True)


def measured_peaks(vr, device):
    """Integer-ALU and L2 peaks of this GPU (vr_probe_peaks), plus MEASURED_PEAKS.json's HBM."""
    import ctypes
    alu, l2 = ctypes.c_double(0), ctypes.c_double(0)
    vr._check(vr.load().vr_probe_peaks(device, ctypes.byref(alu), ctypes.byref(l2)))
    mp = {}
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    return {"alu_tops": alu.value / 1e12, "l2_gbs": l2.value / 1e9, "hbm_gbs": mp.get("hbm_gbs"),
            "source": "alu and l2: measured now by vr_probe_peaks (IMNMX/LOP3 chains; 48 MiB L2-resident re-read); "
                      "hbm: MEASURED_PEAKS.json"}


def ncu_traffic(cfg_name, D, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture
    (profiles/ncu_traffic.json, written by tools/ncu_traffic.py from the capture)."""
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        e = tr[f"{cfg_name}/D{D}"][kernel]
        return e["dram_bytes"], e.get("source")
    except Exception:
        return None, None


def roofline(plan, D, n_steps_dims, peaks, cfg_name):
    """The dominant kernel = the enumeration launch of the dimension with the largest device
    time.  Algorithmic work: rank reads of the candidate examination (a1) +
    (d+1) per scanned cofacet vertex + C(d+2, 2) per tested column (a5); 2 integer ops and 4
    bytes of L2 per read; the (d+1)·⌈log2 n⌉ decode compares are reported as a separate credit
    (the fused kernels never decode)."""
    per = n_steps_dims
    d_star = max(per, key=lambda d: per[d]["ms_enumerate"])
    t = per[d_star]
    ms = t["ms_enumerate"]
    reads = t["reads_a1"] + t["reads_a5"]
    ops = 2.0 * reads
    ops_dec = ops + t["decode"]
    alu_ach = ops / (ms / 1e3) / 1e12
    alu_ach_dec = ops_dec / (ms / 1e3) / 1e12
    l2_ach = 4.0 * reads / (ms / 1e3) / 1e9
    fa, fad, fl = alu_ach / peaks["alu_tops"], alu_ach_dec / peaks["alu_tops"], l2_ach / peaks["l2_gbs"]
    flags = int(t["kernels"])
    kname = ("k_enum_sparse2" if (flags & 4) and d_star >= 2 else "k_enum_sparse") if flags & 4 else \
            ("k_enumerate_flat" if flags & 2 else "k_enumerate")
    kname = f"{kname}<{d_star}>"
    traffic, tsrc = ncu_traffic(cfg_name, D, kname)
    bound = "alu" if fa >= fl else "l2"
    r = {"bound": bound, "kernel": kname, "dimension": d_star,
         "achieved": alu_ach if bound == "alu" else l2_ach, "peak": peaks["alu_tops"] if bound == "alu" else peaks["l2_gbs"],
         "unit": "Tops/s" if bound == "alu" else "GB/s", "frac": fa if bound == "alu" else fl,
         "traffic": traffic, "traffic_unit": "DRAM bytes per launch (ncu --set full, dram__bytes_read + write)",
         "traffic_source": tsrc, "ms_per_launch": ms,
         "alu": {"achieved_tops": alu_ach, "peak_tops": peaks["alu_tops"], "frac": fa,
                 "frac_with_decode_credit": fad, "ops_per_launch": ops, "decode_credit_ops": t["decode"]},
         "l2": {"achieved_gbs": l2_ach, "peak_gbs": peaks["l2_gbs"], "frac": fl, "bytes_per_launch": 4.0 * reads},
         "work": "SURVEY.md 8(d): rank reads = the candidate examination (a1: d per C(n,d+1) index dense; "
                 "output-sensitive: d-1 per C(tau) entry + 1 per (sigma, C(tau) entry), as the kernel reads them) + "
                 "(d+1) per scanned cofacet vertex + C(d+2,2) per tested column (a5); 2 integer ops and 4 B of L2 "
                 "per read; decode compares reported as a credit only",
         "peak_source": peaks["source"]}
    return r


def time_plan(vr, torch, plan, steps, warmup, stream, flush, D, clocks=None):
    """Replays: warm-up, then `steps` timed passes (L2 flushed before each)."""
    for _ in range(warmup):
        plan.replay()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    launches = 0
    stage = {"ms_tables": 0.0, "ms_enumerate": 0.0, "ms_resolve": 0.0, "ms_sort": 0.0}
    dims = {d: None for d in range(1, D + 1)}
    torch.cuda.synchronize()
    for i in range(steps):
        flush.zero_()
        starts[i].record(stream)
        launches += plan.replay()
        ends[i].record(stream)
        tm = plan.timing()  # synchronizes; reads this step's stage events
        for k in stage:
            stage[k] += tm[k] / steps
        for d in range(1, D + 1):
            dt = plan.dim_timing(d)
            if dims[d] is None:
                dims[d] = dict(dt)
                for k in ("ms_enumerate", "ms_resolve", "ms_sort", "ms_setup"):
                    dims[d][k] = 0.0
            for k in ("ms_enumerate", "ms_resolve", "ms_sort", "ms_setup"):
                dims[d][k] += dt[k] / steps
    torch.cuda.synchronize()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    return sum(step_ms) / steps, stage, dims, launches // steps


def e2e_wall(vr, lt_host, n, D, thr, reps, warm=True):
    if warm:
        vr.barcodes(lt_host, n, D, thr)
    walls, bc = [], None
    for _ in range(reps):
        t0 = time.perf_counter()
        bc = vr.barcodes(lt_host, n, D, thr)
        walls.append(time.perf_counter() - t0)
    return statistics.median(walls), bc


def residual_share(bc, D, wall):
    res = sum(bc.stats[d]["ms_residual"] for d in range(1, D + 1)) / 1e3
    cols = sum(bc.stats[d]["residual_columns"] for d in range(1, D + 1))
    surv = sum(bc.stats[d]["survivors"] for d in range(1, D + 1))
    return {"residual_s": res, "share_of_wall": res / wall if wall > 0 else None, "residual_columns": cols,
            "share_of_columns": cols / surv if surv else None, "dim0_s": bc.stats[0]["ms_residual"] / 1e3}


def extra_config(vr, torch, name, stream, flush):
    cfg = G.CONFIGS[name]
    D = cfg.max_dim
    lt_host = torch.from_numpy(cfg.lower_tri()).pin_memory().numpy()
    dev = torch.from_numpy(lt_host).cuda()
    plan = vr.Plan(dev, cfg.n, D, cfg.threshold, stream=stream)
    ms, stage, dims, launches = time_plan(vr, torch, plan, 5, 3, stream, flush, D)
    surv = plan.survivors
    plan.close()
    # (c4b: one call, warmed by the plan's own first run — its host residual takes ~1 min)
    reps = 1 if name == "c4b_torus2000" else 3
    wall, bc = e2e_wall(vr, lt_host, cfg.n, D, cfg.threshold, reps, warm=reps > 1)
    return {"workload": config_obj(cfg, D)["workload"], "survivors": surv, "ms_per_step": ms,
            "value": surv / (ms / 1e3), "unit": UNIT, "stages_ms": stage,
            "dims_ms_enumerate": {d: dims[d]["ms_enumerate"] for d in dims}, "e2e_wall_s": wall,
            "e2e_runs": reps, "residual": residual_share(bc, D, wall), "bars": [len(p) for p in bc.pairs]}


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2502_05063_b200 as vr
    from paper_2502_05063_b200 import build as vrbuild

    if not os.path.exists(vr.lib_path):
        vrbuild.build()
    vr.load()
    torch.cuda.set_device(local_rank)
    cfg, D = workload(args)
    peaks = measured_peaks(vr, local_rank)
    # the input in page-locked host memory (the e2e leg copies it host -> device every call)
    lt_host = torch.from_numpy(cfg.lower_tri()).pin_memory().numpy()
    n = cfg.n
    dev_lt = torch.from_numpy(lt_host).cuda()
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    single = world == 1 and not args.sharded
    dims = None
    if single:
        plan = vr.Plan(dev_lt, n, D, cfg.threshold, stream=stream)
        survivors = plan.survivors
        a_ref = (sum(plan.result.stats[d]["apparent"] for d in range(1, D + 1)),
                 sum(plan.result.stats[d]["residual_columns"] for d in range(1, D + 1)))
        with ClockSampler(local_rank) as clk:
            ms_per_step, stage, dims, launches = time_plan(vr, torch, plan, args.steps, args.warmup, stream, flush, D)
        assert plan.check() == a_ref, "replay did not reproduce the apparent/residual counts"
    else:
        # this rank's shard of every dimension's hot path with the exchanges inside libvr
        # (NCCL: clearing bitmap all-reduce / apparent-cofacet all-gather, residual keys
        # all-gather + device merge); replays time exactly that, max over ranks
        from paper_2502_05063_b200.dist import nccl_comm
        comm = nccl_comm(local_rank)
        plan = vr.Plan(dev_lt, n, D, cfg.threshold, stream=stream, comm=comm)
        survivors = plan.survivors
        for _ in range(args.warmup):
            plan.replay()
        torch.cuda.synchronize()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        launches = 0
        dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local_rank) as clk:
            for i in range(args.steps):
                flush.zero_()
                starts[i].record(stream)
                launches += plan.replay()
                ends[i].record(stream)
            torch.cuda.synchronize()
        dist.barrier()
        ms_local = sum(s.elapsed_time(e) for s, e in zip(starts, ends)) / args.steps
        t = torch.tensor([ms_local], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_per_step = float(t.item())
        launches //= args.steps
        stage = None
    value = survivors / (ms_per_step / 1000.0)  # survivors of the whole (sharded) workload

    # ---- e2e: the public call, H2D of the input and D2H of the barcode in the timed region
    if single:
        e2e_s, bc = e2e_wall(vr, lt_host, n, D, cfg.threshold, args.e2e_steps)
    else:
        from paper_2502_05063_b200.dist import barcodes_comm
        barcodes_comm(lt_host, n, D, cfg.threshold, comm)  # warm
        walls = []
        for _ in range(args.e2e_steps):
            dist.barrier()
            t0 = time.perf_counter()
            bc = barcodes_comm(lt_host, n, D, cfg.threshold, comm)
            walls.append(time.perf_counter() - t0)
        tt = torch.tensor([statistics.median(walls)], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
        plan.close()
        comm.close()
    pairs_bytes = sum(p.nbytes for p in bc.pairs)
    if rank != 0:
        return
    st = bc.stats
    if single:
        roof = roofline(plan, D, dims, peaks, cfg.name)
    else:
        roof = {"bound": None, "kernel": "hot path step (sharded)", "achieved": None, "peak": None, "frac": None,
                "traffic": None, "note": "per-kernel roofline from the single-GPU run"}
    roof["step"] = {"ms_per_step": ms_per_step,
                    "what": "whole hot-path step (tables, every dimension's kernels, sorts, exchanges)"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u32", "data": "synthetic",
        "config": config_obj(cfg, D, {"survivors": survivors,
                                      "parallelism": "single GPU" if single else f"row shards x{world} (NCCL)"}),
        "wall_s": e2e_s,
        "e2e": {"value": survivors / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(lt_host.nbytes),
                "d2h_bytes_per_step": int(pairs_bytes), "wall_s_per_barcode": e2e_s},
        "stages_ms": stage,
        "dims": {d: {k: dims[d][k] for k in ("ms_enumerate", "ms_resolve", "ms_sort", "ms_setup", "survivors")}
                 for d in dims} if dims else None,
        "residual": residual_share(bc, D, e2e_s),
        "columns": {d: {k: st[d][k] for k in ("candidates", "survivors", "apparent", "cleared", "residual_columns",
                                              "queued", "emergent")} for d in range(1, D + 1)},
        "roofline": roof,
        "peaks": peaks,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    # north_star: "next to the paper's quoted Ripser++ speedups with their GPU model (context
    # only)" — PAPER.md Table 5.2, Tesla V100 32 GB + 2x Xeon E5-2680 v4,
    # on the paper's own datasets (ours are synthetic look-alikes of the same n, d)
    line["paper_context"] = {
        "hardware": "Tesla V100 32GB HBM2 + 2x Xeon E5-2680 v4 (PAPER.md P:5741)",
        "table": "PAPER.md Table 5.2 (P:5773-5779): total execution time, Ripser++ vs Ripser",
        "sphere_3_192_d3": {"ripserpp_s": 2.43, "ripser_s": 36.96, "speedup": 15.21},
        "dragon1000_d2": {"ripserpp_s": 5.79, "ripser_s": 48.98, "speedup": 8.46},
        "o3_4096_d3_t1.4": {"ripserpp_s": 11.62, "ripser_s": 64.18, "speedup": 5.52},
    }
    if not args.no_target and single:
        # BASELINE.json north_star target: "the dim-2 n=4096 workload under 1 s on one B200"
        # (reading A22: config 5's O(3)-shaped cloud at max_dim = 2, t = 1.4), end to end
        # through the public host-pointer call
        c5 = G.CONFIGS["c5_o3_4096"]
        lt5 = lt_host if cfg.name == c5.name else c5.lower_tri()
        w5, b5 = e2e_wall(vr, lt5, c5.n, 2, c5.threshold, 3)
        line["target_c5_maxdim2"] = {"wall_s": w5, "target_s": 1.0, "met": w5 < 1.0,
                                     "survivors": sum(b5.stats[d]["survivors"] for d in (1, 2)),
                                     "residual": residual_share(b5, 2, w5), "bars": [len(p) for p in b5.pairs]}
    if single and not args.no_extra:
        line["configs"] = {}
        for name in EXTRA_CONFIGS:
            if name != cfg.name:
                line["configs"][name] = extra_config(vr, torch, name, stream, flush)
    if single and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg, D, args.sample or default_sample(cfg, D))
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"error": str(e)}
    if single and not args.no_ripser:
        try:
            line["cpu_ripser"] = ripser_style_run(cfg, D, bc.threshold, bc.pairs)
        except Exception as e:  # pragma: no cover
            line["cpu_ripser"] = {"error": str(e)}
    print(json.dumps(line), file=OUT, flush=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    global OUT
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run with --gpus ranks
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if args.impl == "ours" and world != args.gpus and not (world == 1 and args.sharded):
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    sys.stdout.flush()
    OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1 or args.sharded:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        dist.init_process_group("nccl", rank=rank, world_size=world)
    run_ours(args, rank, world, local_rank)
    if world > 1 or args.sharded:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

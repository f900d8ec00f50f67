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
Default workload: BASELINE.json configs[1] (n=192 points on S^3, max_dim=3, t = R).

Multi-GPU (torchrun): the workload is sharded over the ranks (strong scaling): every rank
runs its shard of each dimension's hot path, with the two exchanges of SURVEY.md §8(e)
per dimension (clearing-bitmap SUM all-reduce, all-gather of the sorted residual keys) over
NCCL; value = the workload's survivors / max-over-ranks step time.  --impl reference times the
CPU oracle (explicit boundary matrix + Alg 2) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2_s3_192", choices=sorted(G.CONFIGS))
    ap.add_argument("--max-dim", type=int, default=None)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
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


# ------------------------------------------------------------------ CPU oracle baseline
def oracle_sample(cfg, D, m):
    from oracle import oracle as O
    lt = cfg.lower_tri(m)
    t = O.enclosing_radius(lt, m) if math.isinf(cfg.threshold) else cfg.threshold
    t0 = time.perf_counter()
    b = O.barcode(lt, m, D, t)
    dt = time.perf_counter() - t0
    surv = sum(b.n_simplices[1:D + 1])
    return surv, dt


def cpu_baseline(cfg, D, m):
    surv, dt = oracle_sample(cfg, D, m)
    return {"value": surv / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"first {m} points of {cfg.name} (same generator), max_dim={D}, t=R of the sample: "
                      f"{surv} simplices in dims 1..{D}, {dt:.2f} s single-threaded (explicit boundary "
                      f"matrix + standard reduction, no clearing/cohomology/apparent pairs)"}


def ripser_style_run(cfg, D, threshold, gpu_pairs):
    """BASELINE.json north_star: "a single-threaded Ripser-style CPU run timed on the box's
    own host cores in the same run" — cpu_ripser/ (implicit cohomology, clearing, emergent
    pairs, heap columns; §5.2) on the FULL workload at the threshold the GPU path
    used, its bars compared with the GPU path's."""
    import cpu_ripser as RS
    RS.build()
    lt = cfg.lower_tri()
    t0 = time.perf_counter()
    pairs, st = RS.barcode(lt, cfg.n, D, threshold)
    dt = time.perf_counter() - t0
    surv = sum(st[d]["simplices"] for d in range(1, D + 1))

    def srt(a):
        a = np.asarray(a, np.float32).reshape(-1, 2)
        return a[np.lexsort((a[:, 1], a[:, 0]))] if len(a) else a
    same = all(np.array_equal(srt(pairs[d]), srt(gpu_pairs[d])) for d in range(D + 1))
    return {"value": surv / dt, "unit": UNIT, "cores": 1, "kind": "ripser-style", "wall_s": dt,
            "bars_equal_gpu": bool(same),
            "per_dim_ms": [round(s["ms"], 1) for s in st],
            "sample": f"full {cfg.name} workload, max_dim={D}, t={threshold:.6g}: {surv} simplices in dims 1..{D}, "
                      f"single-threaded cpu_ripser (implicit coboundary cohomology + clearing + emergent pairs)"}


def default_sample(cfg, D):
    return {1: 64, 2: 64, 3: 56}.get(D, 40) if cfg.n > 64 else cfg.n


# ------------------------------------------------------------------ arms
def run_reference(args, rank, world):
    cfg, D = workload(args)
    if rank != 0:
        return
    m = args.sample or {1: 64, 2: 48, 3: 48}.get(D, 32)
    m = min(m, cfg.n)
    from oracle import oracle as O
    O.build()
    for _ in range(args.warmup):
        oracle_sample(cfg, D, m)
    tot_s, tot_t = 0, 0.0
    for _ in range(args.steps):
        s, dt = oracle_sample(cfg, D, m)
        tot_s += s
        tot_t += dt
    v = tot_s / tot_t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * tot_t / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_obj(cfg, D, {"sample_points": m}),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"first {m} points of {cfg.name} per step, max_dim={D}"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), file=OUT, flush=True)


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
    # the input in page-locked host memory (the e2e leg copies it host -> device every call)
    lt_host = torch.from_numpy(cfg.lower_tri()).pin_memory().numpy()
    n = cfg.n
    dev_lt = torch.from_numpy(lt_host).cuda()
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    if world == 1 and not args.sharded:
        plan = vr.Plan(dev_lt, n, D, cfg.threshold, stream=stream)
        survivors = plan.survivors
        step_fn = plan.replay
        a_ref = (sum(plan.result.stats[d]["apparent"] for d in range(1, D + 1)),
                 sum(plan.result.stats[d]["residual_columns"] for d in range(1, D + 1)))
    else:
        # shards of every dimension's hot path + the two exchanges per dimension (NCCL)
        from paper_2502_05063_b200.dist import ShardedHotPath
        plan = ShardedHotPath(dev_lt, n, D, cfg.threshold)
        survivors = plan.survivors_total
        step_fn = plan.step
        a_ref = None

    for _ in range(args.warmup):
        step_fn()
    torch.cuda.synchronize()
    if a_ref is not None:
        assert plan.check() == a_ref, "replay did not reproduce the apparent/residual counts"

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches = 0
    stage = {"ms_tables": 0.0, "ms_enumerate": 0.0, "ms_resolve": 0.0, "ms_sort": 0.0}
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(stream)
            launches += step_fn()
            ends[i].record(stream)
            if a_ref is not None:
                tm = plan.timing()  # synchronizes; reads this step's stage events
                for k in stage:
                    stage[k] += tm[k]
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    if a_ref is not None:
        assert plan.check() == a_ref
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms_max = float(t.item())
    ms_per_step = total_ms_max / args.steps
    value = survivors / (ms_per_step / 1000.0)  # survivors of the whole (sharded) workload

    # ---- e2e: the public call, H2D of the input and D2H of the barcode in the timed region
    e2e_times, pairs_bytes = [], 0

    def e2e_call():
        if a_ref is not None:
            return vr.barcodes(lt_host, n, D, cfg.threshold)
        from paper_2502_05063_b200.dist import barcodes_sharded
        return barcodes_sharded(torch.from_numpy(lt_host).cuda(non_blocking=True), n, D, cfg.threshold)

    e2e_call()  # warm
    for _ in range(args.e2e_steps):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        bc = e2e_call()
        e2e_times.append(time.perf_counter() - t0)
        pairs_bytes = sum(p.nbytes for p in bc.pairs)
    e2e_s = statistics.median(e2e_times)
    tt = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e_s = float(tt.item())
    st = bc.stats

    if rank != 0:
        return
    if a_ref is None:  # per-stage device times are reported by the single-GPU replay only
        tm = {"rank_ops_enumerate": 0.0, "rank_ops_resolve": 0.0}
    else:
        tm = plan.timing()
    # the workload's method-level op count — a property of the workload, not of
    # the sharding (the shards partition the candidates; every candidate's scan is its own):
    # from an UNTIMED single-GPU plan of the same input when the timed path is sharded
    if a_ref is not None:
        ops_total = tm["rank_ops_enumerate"] + tm["rank_ops_resolve"]
    else:
        p1 = vr.Plan(dev_lt, n, D, cfg.threshold, stream=stream)
        t1 = p1.timing()
        ops_total = t1["rank_ops_enumerate"] + t1["rank_ops_resolve"]
        p1.close()
    per = {k: stage[k] / args.steps for k in stage}
    # roofline of the dominant kernel: k_enumerate is ALU-bound —
    # algorithmic work = SURVEY.md 8(d)'s integer-op figure (computed by the library);
    # peak = 148 SMs x 4 SMSPs x 16 lanes/clk (ALU pipe, IMNMX/ISETP) x measured max SM clock.
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    alu_peak = 148 * 4 * 16 * sm_mhz * 1e6 / 1e12  # T int-ops/s
    # both hot kernels are gathers over the L2-resident rank matrix followed by integer
    # max/compare chains; their algorithmic work is the method's rank comparisons
    kern = {
        "k_enumerate": (tm["rank_ops_enumerate"], per["ms_enumerate"]),
        "k_resolve": (tm["rank_ops_resolve"], per["ms_resolve"]),
    }
    dom = max(kern, key=lambda k: kern[k][1])
    ops, ms = kern[dom]
    achieved = ops / (ms / 1000.0) / 1e12 if ms > 0 else None
    traffic = None
    try:  # DRAM bytes per step of the dominant kernel, from the committed ncu full capture
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        if dom in tr and cfg.name == "c2_s3_192" and D == 3:
            traffic = sum(tr[dom].values())
    except Exception:
        pass
    roof = {"bound": "alu", "kernel": dom, "achieved": achieved, "peak": alu_peak, "unit": "Tops/s",
            "frac": (achieved / alu_peak) if achieved else None, "traffic": traffic,
            "traffic_unit": "DRAM bytes per step (all launches of the kernel), ncu --set full capture",
            "ops_per_step": ops, "ms_per_step": ms,
            "all": {k: {"ops": o, "ms": m, "tops": (o / (m / 1000.0) / 1e12) if m > 0 else None}
                    for k, (o, m) in kern.items()},
            "peak_source": "derived: 148 SM x 64 ALU lanes/clk x sm_max_mhz (MEASURED_PEAKS.json); "
                           "work = SURVEY.md 8(d) per-unit figures: 2 integer ops per rank read (d per candidate, "
                           "(d+1) per scanned cofacet vertex, C(d+2,2) per tested column) + (d+1)*ceil(log2 n) "
                           "decode compares per tested column"}
    # step-level roofline at every N: the workload's rank ops over the WHOLE step time (all
    # kernels, sort and exchanges included) against N GPUs' ALU peak — a lower bound on the
    # dominant kernel's fraction, and the number that stays defined for the sharded path
    step_ach = ops_total / (ms_per_step / 1000.0) / 1e12 if ms_per_step > 0 else None
    roof["step"] = {"achieved": step_ach, "peak": alu_peak * world, "unit": "Tops/s",
                    "frac": (step_ach / (alu_peak * world)) if step_ach else None, "ops_per_step": ops_total,
                    "what": "workload rank ops / whole hot-path step time, vs n_gpus x ALU peak"}
    if a_ref is None:  # sharded: no per-kernel events; the step-level figure is the roofline
        roof.update({"kernel": "hot path step (sharded)", "achieved": step_ach, "peak": alu_peak * world,
                     "frac": roof["step"]["frac"], "ops_per_step": ops_total, "ms_per_step": ms_per_step})
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u32", "data": "synthetic",
        "config": config_obj(cfg, D, {"survivors": survivors,
                                      "parallelism": "single GPU" if a_ref is not None else f"row shards x{world}"}),
        "wall_s": e2e_s,
        "e2e": {"value": survivors / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(lt_host.nbytes),
                "d2h_bytes_per_step": int(pairs_bytes), "wall_s_per_barcode": e2e_s},
        "stages_ms": per,
        "residual_ms": sum(st[d]["ms_residual"] for d in range(1, D + 1)),
        "dim0_ms": st[0]["ms_residual"],
        "columns": {d: {k: st[d][k] for k in ("candidates", "survivors", "apparent", "cleared", "residual_columns",
                                              "queued", "emergent")} for d in range(1, D + 1)},
        "roofline": roof,
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
    if not args.no_target and world == 1:
        # BASELINE.json north_star target: "the dim-2 n=4096 workload under 1 s on one B200"
        # (reading A22: config 5's o3-shaped cloud at max_dim = 2, t = 1.4), end to end
        # through the public host-pointer call
        c5 = G.CONFIGS["c5_o3_4096"]
        lt5 = c5.lower_tri()
        vr.barcodes(lt5, c5.n, 2, c5.threshold)  # warm
        walls = []
        for _ in range(3):
            t0 = time.perf_counter()
            b5 = vr.barcodes(lt5, c5.n, 2, c5.threshold)
            walls.append(time.perf_counter() - t0)
        line["target_c5_maxdim2"] = {"wall_s": statistics.median(walls), "target_s": 1.0,
                                     "survivors": sum(b5.stats[d]["survivors"] for d in (1, 2)),
                                     "bars": [len(p) for p in b5.pairs]}
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg, D, args.sample or default_sample(cfg, D))
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"error": str(e)}
        try:
            line["cpu_ripser"] = ripser_style_run(cfg, D, bc.threshold, bc.pairs)
        except Exception as e:  # pragma: no cover
            line["cpu_ripser"] = {"error": str(e)}
    print(json.dumps(line), file=OUT, flush=True)


def main():
    global OUT
    args = parse()
    sys.stdout.flush()
    OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    world = int(os.environ.get("WORLD_SIZE", "1"))
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
        os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group("nccl", rank=rank, world_size=world)
    run_ours(args, rank, world, local_rank)
    if world > 1 or args.sharded:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

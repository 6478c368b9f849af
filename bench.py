#!/usr/bin/env python
"""Benchmark of the chemistry hot path on B200: chemistry Mcell-steps/s (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

A "step" is one pass of the whole hot path (gate -> bulk bursts ->
compaction -> sparse -> write-back, one fused chem_integrate_boxes call over every box of the
field) over one batch of synthetic input: one CFD dt of every cell.  One cell-step = one cell
advanced over one dt.  Inputs are restored from a pristine device copy before each
step (untimed).  value = cells of all ranks / (max over ranks of the CUDA-event step time).

Multi-GPU: cells are independent 0-D reactors, so every rank integrates its own
field (weak scaling) with no data-path collective; NCCL carries only the max-time reduction.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

RTOL, ATOL, ATOL_T = 1e-9, 1e-20, 1e-6        # parity tolerance (headline measured there)
METRIC = "chemistry Mcell-steps/s per B200 at 1/2/4/8 GPUs; % of FP64/HBM roofline"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="cfg2")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--rtol", type=float, default=RTOL)
    p.add_argument("--atol", type=float, default=ATOL)
    p.add_argument("--method", default="rodas4", choices=["rodas4", "rodas3", "explicit", "ros4"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-sample-seconds", type=float, default=15.0)
    p.add_argument("--balance", default="lpt", choices=["lpt", "none"])
    p.add_argument("--lanes", type=int, default=1, choices=[1, 4, 8], help="lanes per cell (1: thread per cell)")
    p.add_argument("--tmode", type=int, default=0, choices=[0, 1],
                   help="0: T integrated by Eq. 6; 1: T = Newton(e, Y) at every RHS evaluation (P:96)")
    p.add_argument("--e2e-chunks", type=int, default=0, help="e2e copy/compute pipelining groups (0: auto)")
    p.add_argument("--h0", type=float, default=0.01, help="initial substep factor (chem_opts.h0_factor)")
    p.add_argument("--opt", action="append", default=[], metavar="KEY=VAL",
                   help="extra chem_opts field (e.g. kmax_bulk=5, refill_bulk=1); repeatable")
    p.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                   help="process-group backend (gloo only to exercise N>1 on a box with fewer GPUs)")
    return p.parse_args()


# ------------------------------------------------------------------ clocks during the timed region
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, pw, reasons = [], [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0])); mx.append(float(parts[1])); pw.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [s for s, p in zip(sm, pw)] if sm else []
        return {"sm_mhz": float(np.median(load)) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None, "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------------ workloads
class Workload:
    """boxes (this rank's), the fused calls one step makes (lists of box indices), pristine inputs."""

    def __init__(self, boxes, calls, meta, cell_steps, extra=None):
        import torch
        self.boxes, self.calls, self.meta = boxes, calls, meta
        self.cell_steps = cell_steps                 # cell-steps this rank advances per step
        self.pristine = [(b.T.clone(), b.Y.clone()) for b in boxes]
        self.extra = extra or {}
        torch.cuda.synchronize()

    def restore(self):
        for b, (T, Y) in zip(self.boxes, self.pristine):
            b.T.copy_(T)
            b.Y.copy_(Y)

    def step(self, chem, rtol, atol, cost=None):
        stats = []
        for c in self.calls:
            bx = [self.boxes[i] for i in c]
            cc = None
            if cost is not None:
                import torch
                cc = torch.zeros(len(c), dtype=torch.float64, device=self.boxes[0].rho.device)
            stats.append(chem.integrate_boxes(bx, rtol=rtol, atol=atol, box_cost=cc))
            if cost is not None:
                cost[c] += cc.cpu().numpy()
        return stats


def _mk_boxes(chem, raw):
    from paper_2510_23993_b200 import Box
    out = []
    for b in raw:
        e = chem.energy(b["T"], b["Y"])            # e = u(T0, Y) with the CUDA path's own thermo
        out.append(Box(b["rho"], e, b["T"].clone(), b["Y"].clone(), b["dt"], b.get("solid")))
    return out


def build_workload(args, chem, doc, device, rank, world):
    import synth
    from paper_2510_23993_b200 import sharding
    m = chem.mech
    if args.config == "cfg2":
        raw, meta = synth.field_cfg2(doc, device=device)
        boxes = _mk_boxes(chem, raw)
        return Workload(boxes, [list(range(len(boxes)))], meta, sum(b.ncells for b in boxes))
    if args.config == "cfg3":
        raw, meta = synth.field_cfg3(doc, m.W, m.species, device=device)
        boxes = _mk_boxes(chem, raw)
        return Workload(boxes, [list(range(len(boxes)))], meta, sum(b.ncells for b in boxes))
    if args.config == "cfg5":
        nb = 128
        ids = list(range(rank, nb, world))         # strong split of one field over the ranks
        raw, meta = synth.field_cfg5(doc, m.W, m.species, device=device, box_ids=ids)
        boxes = _mk_boxes(chem, raw)
        meta["scaling"] = "strong"
        return Workload(boxes, [list(range(len(boxes)))], meta, sum(b.ncells for b in boxes))
    if args.config == "cfg4":
        # weak scaling: P copies of the 3-level hierarchy; copy p calibrated on rank p, then the
        # P*192 boxes are redistributed by LPT on the measured per-box cost.
        import numpy as np
        all_desc = [d for p in range(world) for d in synth.hierarchy_cfg4(copy=p)]
        mine = [i for i, d in enumerate(all_desc) if d["copy"] == rank]

        def calls_for(idx):
            lv = [all_desc[i]["level"] for i in idx]
            # one coarse step with subcycling: L0 x1 (dt), L1 x2 (dt/2), L2 x4 (dt/4),
            # fused across levels: {L0,L1,L2}, {L1,L2}, {L2}, {L2}
            return [[k for k, l in enumerate(lv) if l >= 0], [k for k, l in enumerate(lv) if l >= 1],
                    [k for k, l in enumerate(lv) if l >= 2], [k for k, l in enumerate(lv) if l >= 2]]

        raw = [synth.build_cfg4_box(doc, m.W, m.species, all_desc[i], device) for i in mine]
        w0 = Workload(_mk_boxes(chem, raw), calls_for(mine), {}, 0)
        cost = np.zeros(len(mine))
        w0.step(chem, args.rtol, args.atol, cost=cost)
        if world > 1 and args.balance == "lpt":
            gcost, owner = sharding.balance(cost)
        else:
            gcost = np.concatenate([cost] * world) if world > 1 else cost
            owner = np.array([d["copy"] for d in all_desc])
        imb = sharding.imbalance(gcost, owner, world) if world > 1 else 1.0
        own = [i for i in range(len(all_desc)) if owner[i] == rank]
        if own == mine:
            boxes = w0.boxes
        else:
            del w0
            boxes = _mk_boxes(chem, [synth.build_cfg4_box(doc, m.W, m.species, all_desc[i], device) for i in own])
        calls = calls_for(own)
        cell_steps = sum(b.ncells * 2 ** all_desc[i]["level"] for b, i in zip(boxes, own))
        meta = dict(workload=f"cfg4: 3-level AMR hierarchy (ratio 2, 32^3 boxes, 192 boxes/copy, 6.3M cells/copy) "
                             f"of detonation fields, {world} copies, subcycled coarse step (4 fused calls), "
                             f"balance={args.balance}", cells=sum(b.ncells for b in boxes))
        return Workload(boxes, calls, meta, cell_steps, extra=dict(imbalance_max_over_mean=imb,
                                                                   boxes_owned=len(own)))
    raise SystemExit(f"unknown --config {args.config}")


# ------------------------------------------------------------------ oracle (cpu baseline / reference arm)
def oracle_sample(meta, seconds_target, rtol, atol):
    """Time the oracle, as it stands, on a bounded sample of the workload's cells (all host cores)."""
    from oracle import Oracle
    o = Oracle("h2air_li2004")
    st = meta["state"]
    Y = np.asarray(st["Y"])
    e = o.energy(st["T"], Y)
    nth = o.max_threads()

    def run(n):
        t0 = time.perf_counter()
        o.integrate_cells(np.full(n, st["rho"]), np.full(n, e), np.full(n, st["T"]), np.tile(Y, (n, 1)), 1e-7,
                          rtol=rtol, atolY=atol, atolT=ATOL_T, nthreads=nth)
        return time.perf_counter() - t0

    n = nth
    dt = run(n)
    while dt < 0.5 and n < 1 << 22:         # calibrate the sample to ~seconds_target of CPU work
        n *= 4
        dt = run(n)
    n = int(max(nth, min(1 << 24, n * seconds_target / max(dt, 1e-9))))
    dt = run(n)
    return dict(cells=n, seconds=dt, threads=nth, value=n / dt / 1e6)


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synth
    doc = synth.load_trajectories()
    if args.config != "cfg2":
        print(json.dumps({"impl": "reference", "unavailable": "reference arm implemented for cfg2 only"}))
        return
    meta = _meta_cfg2(doc)
    times, cells = [], 0
    for i in range(args.warmup + args.steps):
        r = oracle_sample(meta, max(2.0, min(20.0, 60.0 / max(1, args.steps))), args.rtol, args.atol)
        if i >= args.warmup:
            times.append(r["seconds"])
            cells += r["cells"]
            nth = r["threads"]
    value = cells / sum(times) / 1e6
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "Mcell-steps/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": meta["workload"], "rtol": args.rtol, "atol_Y": args.atol, "atol_T": ATOL_T},
            "cpu_baseline": {"value": value, "unit": "Mcell-steps/s", "cores": nth, "kind": "oracle",
                             "sample": f"{cells // args.steps} cells of the {args.config} state per step "
                                       "(all cells of cfg2 are identical)"},
            "e2e": {"value": value, "unit": "Mcell-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def _meta_cfg2(doc):
    import synth
    tr = next(t for t in doc["trajectories"] if t["kind"] == "fresh" and t["T0"] == 1200.0)
    rho, T, Y = synth.traj_state(tr, 0.9)
    return dict(workload="cfg2: uniform 128^3 H2-air field, T0=1200 K traj. state at t=0.9 tau, 64 boxes of 32^3, "
                         "dt=1e-07 s", cells=128 ** 3, state=dict(rho=float(rho), T=float(T), Y=np.asarray(Y).tolist()))


# ------------------------------------------------------------------ our arm
def oracle_sample_field(wl, seconds_target, rtol, atol, T_min=500.0):
    """cpu_baseline for a non-uniform field: the oracle on a random sample of the field's active
    cells (each rank-0 box contributes), extrapolated to the field as n_active x (time per sampled
    cell with all threads); gated cells cost nothing on either side.  Labelled an extrapolation."""
    import torch
    from oracle import Oracle
    o = Oracle("h2air_li2004")
    rng = np.random.default_rng(0)
    cells, n_act = [], 0
    for bi, (b, (T0, Y0)) in enumerate(zip(wl.boxes, wl.pristine)):
        act = np.nonzero((T0 >= T_min).cpu().numpy())[0]
        n_act += len(act)
        if not len(act):
            continue
        pick = np.sort(rng.choice(act, size=min(len(act), 8192), replace=False))
        idx = torch.as_tensor(pick, device=b.rho.device)
        rho_b, T_b, Y_b = b.rho[idx].cpu().numpy(), T0[idx].cpu().numpy(), Y0[:, idx].cpu().numpy().T
        cells.extend(zip(rho_b, T_b, Y_b, [b.dt] * len(pick)))
    rng.shuffle(cells)
    nth = o.max_threads()

    def run(sub):
        rho = np.array([c[0] for c in sub]); T = np.array([c[1] for c in sub]); Y = np.array([c[2] for c in sub])
        e = np.array([o.energy(t, y) for t, y in zip(T, Y)])
        t0 = time.perf_counter()
        for d in sorted(set(c[3] for c in sub)):
            sel = np.array([c[3] == d for c in sub])
            o.integrate_cells(rho[sel], e[sel], T[sel], Y[sel], d, rtol=rtol, atolY=atol, atolT=ATOL_T, nthreads=nth)
        return time.perf_counter() - t0

    n = min(len(cells), 4 * nth)
    dt = run(cells[:n])
    while dt < seconds_target / 2 and n < len(cells):
        n = min(len(cells), n * 4)
        dt = run(cells[:n])
    per_cell = dt / n
    total_cells = sum(b.ncells for b in wl.boxes)
    value = total_cells / (n_act * per_cell) / 1e6
    return dict(value=value, threads=nth, cells=n, seconds=dt, n_active=n_act,
                sample=f"{n} random active cells of the {wl.meta['workload'][:5]} field timed on {nth} threads "
                       f"({dt:.1f} s), extrapolated to the field's {n_act} active of {total_cells} cells")


def ours(args):
    import torch
    import torch.distributed as dist

    import synth
    from paper_2510_23993_b200 import Chem
    from paper_2510_23993_b200.api import HostRunner
    from paper_2510_23993_b200.flops import FlopModel, fp64_peak_tflops

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group("gloo")
    method = {"rodas4": 0, "rodas3": 1, "explicit": 2, "ros4": 3}[args.method]
    chem = Chem("h2air_li2004", device=local, atol_T=ATOL_T, method=method, lanes_per_cell=args.lanes,
                temperature_mode=args.tmode, h0_factor=args.h0,
                **{k: float(v) if "." in v or "e" in v else int(v) for k, v in (o.split("=", 1) for o in args.opt)})
    doc = synth.load_trajectories()
    wl = build_workload(args, chem, doc, device, rank, world)
    ncells = sum(b.ncells for b in wl.boxes)
    fm = FlopModel(chem.mech, stages={0: 6, 1: 4, 2: 0, 3: 4}[method])

    for _ in range(args.warmup):
        wl.restore()
        wl.step(chem, args.rtol, args.atol)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    stats = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    for k in range(args.steps):
        wl.restore()                                   # untimed: before the start event
        ev[k][0].record()
        stats += wl.step(chem, args.rtol, args.atol)
        ev[k][1].record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_total = sum(step_ms) / 1e3
    t_rank = t_total
    tot_cs = wl.cell_steps
    if world > 1:
        from paper_2510_23993_b200 import sharding
        t_total = float(sharding.reduce_stats([t_total], "max")[0])          # max over ranks
        tot_cs = float(sharding.reduce_stats([float(wl.cell_steps)], "sum")[0])
    value = tot_cs * args.steps / t_total / 1e6

    # roofline of the dominant kernel (k_integrate: bulk + sparse launches, CUDA-event timed by the
    # library on the launching stream)
    flops = sum(fm.flops(s) for s in stats)
    k_ms = sum(s["t_bulk_ms"] + s["t_sparse_ms"] for s in stats)
    launches_int = sum(s["bulk_iters"] + (1 if s["sparse_cells"] > 0 else 0) for s in stats)
    achieved = flops / (k_ms / 1e3) / 1e12 if k_ms > 0 else 0.0
    sm_mhz_peak = 1965.0
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        sm_mhz_peak = float(mp.get("sm_max_mhz", sm_mhz_peak))
    except Exception:
        pass
    peak = fp64_peak_tflops(sm_mhz=sm_mhz_peak)
    gpu_launches = sum(1 + 2 * s["bulk_iters"] + (1 if s["sparse_cells"] > 0 else 0) for s in stats)
    traffic, ncu_pipe = None, None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(args.config)
        if tr:
            traffic, ncu_pipe = tr["traffic_bytes_per_launch"], tr.get("ncu_fp64_pipe_pct")
    except Exception:
        pass

    # e2e through the public API with host buffers (H2D + calls + D2H inside the timed region)
    e2e = None
    if not args.no_e2e:
        host = [dict(rho=b.rho.cpu().pin_memory(), e=b.e.cpu().pin_memory(), T=p[0].cpu().pin_memory(),
                     Y=p[1].cpu().pin_memory(), dt=b.dt) for b, p in zip(wl.boxes, wl.pristine)]
        # copy/compute pipelining pays on dense fields; on sparse ones (cfg3/cfg4) splitting the fused
        # call serialises the chunks' long tails, so those run as one call
        chunks = args.e2e_chunks if args.e2e_chunks > 0 else (5 if args.config in ("cfg2", "cfg5") else 1)
        hr = HostRunner(chem, host, wl.calls, chunks=chunks)
        hr.step(args.rtol, args.atol)
        torch.cuda.synchronize()
        e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(args.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            e_ev[k][0].record()
            hr.step(args.rtol, args.atol)
            e_ev[k][1].record()
        torch.cuda.synchronize()
        te = sum(a.elapsed_time(b) for a, b in e_ev) / 1e3
        if world > 1:
            from paper_2510_23993_b200 import sharding
            te = float(sharding.reduce_stats([te], "max")[0])
        e2e = {"value": tot_cs * args.steps / te / 1e6, "unit": "Mcell-steps/s",
               "h2d_bytes_per_step": hr.h2d_bytes, "d2h_bytes_per_step": hr.d2h_bytes,
               "copy_compute_chunks": chunks if hr.pipelined else 1}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if args.config == "cfg2":
            r = oracle_sample(wl.meta, args.cpu_sample_seconds, args.rtol, args.atol)
            cpu = {"value": r["value"], "unit": "Mcell-steps/s", "cores": r["threads"], "kind": "oracle",
                   "sample": f"{r['cells']} cells of the cfg2 state (all cfg2 cells are identical), "
                             f"{r['seconds']:.1f} s on {r['threads']} threads, same rtol/atol as the GPU run"}
        else:
            r = oracle_sample_field(wl, args.cpu_sample_seconds, args.rtol, args.atol)
            cpu = {"value": r["value"], "unit": "Mcell-steps/s", "cores": r["threads"], "kind": "oracle",
                   "sample": r["sample"], "extrapolated": True}

    att = sum(s["steps_attempted"] for s in stats) / args.steps
    acc = sum(s["steps_accepted"] for s in stats) / args.steps
    s0 = stats[-1]
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Mcell-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_total / args.steps, "higher_is_better": True,
            "scaling": wl.meta.get("scaling", "weak"), "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl.meta["workload"], "cells_per_gpu": ncells, "boxes_per_gpu": len(wl.boxes),
                       "cell_steps_per_step_per_gpu": wl.cell_steps, "fused_calls_per_step": len(wl.calls),
                       "rtol": args.rtol, "atol_Y": args.atol, "atol_T": ATOL_T, "method": args.method,
                       "lanes_per_cell": args.lanes, "temperature_mode": args.tmode, "h0_factor": args.h0,
                       **({"opts": args.opt} if args.opt else {}),
                       "l2": "inputs >= 369 MB/GPU > 126 MB L2 (no flush needed)",
                       "parallelism": f"boxes over {world} rank(s)",
                       "schedule": {1: "heavy-first (cost hints: the previous step's per-cell substeps; "
                                       "the warm-up steps seed them)",
                                    2: "bulk-sparse (Alg. 3), bulk list sorted by the previous step's "
                                       "per-cell substeps"}.get(s0.get("lpt", 0), "bulk-sparse (Alg. 3)"),
                       **wl.extra},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_unit": "bytes per launch (ncu)",
                         "ncu_fp64_pipe_pct": ncu_pipe,
                         "kernel": "k_integrate (bulk+sparse)", "flops_per_step_model": fm.per_step(),
                         "peak_source": "148 SMs x 64 FP64 FMA/clk x 2 x sm_max_mhz (derived, DESIGN.md)"},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": gpu_launches, "clocks": clk,
            "detail": {"step_ms": step_ms, "rank0_seconds": t_rank, "k_integrate_ms": k_ms / args.steps,
                       "integrate_launches": launches_int, "substeps_per_cell_step": att / max(wl.cell_steps, 1),
                       "accepted_per_cell_step": acc / max(wl.cell_steps, 1),
                       "frozen_per_cell_step": sum(s.get("steps_frozen", 0) for s in stats) / args.steps
                       / max(wl.cell_steps, 1), "bulk_iters": s0["bulk_iters"],
                       "active_per_iter": s0["active_per_iter"], "sparse_cells": s0["sparse_cells"],
                       "active0": s0["active0"], "t_gate_ms": s0["t_gate_ms"], "t_compact_ms": s0["t_compact_ms"],
                       "t_sparse_ms": s0["t_sparse_ms"], "n_unfinished": s0["n_unfinished"],
                       "n_nonfinite": s0["n_nonfinite"], "max_energy_drift": s0["max_energy_drift"],
                       "lockstep": s0["lockstep"], "lpt": s0.get("lpt", 0),
                       "bulk_simt_eff": s0["bulk_substeps"] / max(32 * s0["warp_substeps"], 1)},
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()

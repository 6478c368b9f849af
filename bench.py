#!/usr/bin/env python
"""Benchmark of the chemistry hot path on B200: chemistry Mcell-steps/s (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

A "step" is one pass of the whole hot path (gate -> bulk bursts ->
compaction -> sparse -> write-back, fused chem_integrate_boxes calls over every box of the field)
over one batch of synthetic input: one CFD dt of every cell.  One cell-step = one cell advanced over
one dt.  value = cells of all ranks / (max over ranks of the CUDA-event step time).

Inputs between timed steps (untimed, before the start event) — VERDICT r01 next-4:
  * cfg2 (every cell the same state by definition): restored from the pristine copy;
  * cfg3/cfg4/cfg5 ("shift", default): the pristine field advanced by one cell along x per step
    (step k = the field rolled by k cells along x inside every box), the way a front moves through
    the grid of a CFD run: every step integrates the same multiset of states (the named config),
    but the previous step's per-cell substep counts, the heavy-first schedule's cost hints, sit
    one cell behind the cells they describe - a prediction, not a replay.  ("perturb": a seeded
    +-1 % T jitter with e recomputed, which knocks burnt cells off equilibrium and so inflates
    the work; kept as an option.)  The line also reports the first call of a layout (no cost
    hints), Alg. 3 as written (schedule_lpt = 0) and exact replay (restore), timed the same way.
With no flags (the driver's command) the cfg2 headline line carries, under "also", the cfg2b variant
(t/tau ~ U[0.85, 0.95] per cell) and the cfg3 bulk-sparse field timed under Alg. 3 and under the
default schedule, so the driver measures intra-warp divergence and a non-empty sparse phase.

Multi-GPU: cells are independent 0-D reactors, so every rank integrates its own
boxes with no data-path collective.  NCCL carries the cost all_gather of the LPT balance (cfg4,
cfg5) and, every step, the SUM of unfinished cells / substeps and the MIN of the proposed dt.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

RTOL, ATOL, ATOL_T = 1e-9, 1e-20, 1e-6        # parity tolerance (headline measured there)
PROD_TOL = dict(rtol=1e-6, atol=1e-12, atol_T=1e-3)   # §8(d) secondary production-tolerance number
METRIC = "chemistry Mcell-steps/s per B200 at 1/2/4/8 GPUs; % of FP64/HBM roofline"
T_MIN = 500.0
METHODS = {"rodas4": 0, "rodas3": 1, "explicit": 2}
STAGES = {0: 6, 1: 4, 2: 0}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="cfg2")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--rtol", type=float, default=RTOL)
    p.add_argument("--atol", type=float, default=ATOL)
    p.add_argument("--method", default="rodas4", choices=list(METHODS))
    p.add_argument("--mech", default="h2air_li2004",
                   help="mechanism (mech/<name>.yaml); fields of the 9 H2-air species are mapped by name, "
                        "NO at 100 ppm by mass replacing N2 when the mechanism has it (NEXT-3)")
    p.add_argument("--evolve", default="auto", choices=["auto", "shift", "perturb", "restore"],
                   help="inputs between steps (auto: restore for cfg2, shift otherwise)")
    p.add_argument("--perturb", type=float, default=0.01, help="relative T jitter of --evolve perturb")
    p.add_argument("--also", default="auto",
                   help="extra configs timed into the same line ('auto': cfg2b and cfg3 when --config cfg2; 'none')")
    p.add_argument("--no-schedules", action="store_true", help="skip the first-call / alg3 / replay variants")
    p.add_argument("--no-prod", action="store_true", help="skip the production-tolerance number")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-sample-seconds", type=float, default=15.0)
    p.add_argument("--balance", default="lpt", choices=["lpt", "none"])
    p.add_argument("--e2e-chunks", type=int, default=0, help="e2e copy/compute pipelining groups (0: auto)")
    p.add_argument("--e2e-taper", type=float, default=2.0,
                   help="e2e: share of a middle group relative to the first and last groups")
    p.add_argument("--opt", action="append", default=[], metavar="KEY=VAL",
                   help="extra chem_opts field (e.g. kmax_bulk=5, schedule_lpt=0); repeatable")
    p.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                   help="process-group backend (gloo only to exercise N>1 on a box with fewer GPUs)")
    return p.parse_args()


def _opts(args):
    return {k: float(v) if ("." in v or "e" in v) else int(v) for k, v in (o.split("=", 1) for o in args.opt)}


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
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self, min_samples=3, wait_s=2.0):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t0 = time.time()
        while len(self.lines) < min_samples and time.time() - t0 < wait_s:   # short regions: wait for samples
            time.sleep(0.02)
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
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None, "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------------ workloads
class Workload:
    """boxes (this rank's), the fused calls one step makes (lists of box indices), pristine inputs,
    and the per-step input preparation (restore or seeded perturbation; untimed)."""

    def __init__(self, chem, boxes, calls, meta, cell_steps, evolve, amp, extra=None):
        import torch
        self.chem = chem
        self.boxes, self.calls, self.meta = boxes, calls, meta
        self.cell_steps = cell_steps                 # cell-steps this rank advances per step
        self.pristine = [(b.T.clone(), b.Y.clone(), b.e.clone()) for b in boxes]
        self.active = [T >= T_MIN for T, _, _ in self.pristine]
        self.evolve, self.amp = evolve, amp
        self.rho0 = [b.rho.clone() for b in boxes]
        self.solid0 = [b.solid.clone() if b.solid is not None else None for b in boxes]
        if evolve == "shift":
            # boxes are cubes, x fastest: roll along x inside each box
            self.box_nx = [round(b.ncells ** (1 / 3)) for b in boxes]
            assert all(n ** 3 == b.ncells for n, b in zip(self.box_nx, boxes)), "shift needs cubic boxes"
        self.extra = extra or {}
        self.ncells = sum(b.ncells for b in boxes)
        torch.cuda.synchronize()

    def prepare(self, k):
        """Inputs of step k: the pristine field; (shift) rolled by k cells along x inside every box;
        (perturb) its active cells' T jittered by a seeded +-amp that differs for every k (cells stay
        active), e = u(T', Y) by chem_energy."""
        import torch
        for i, (b, (T, Y, e)) in enumerate(zip(self.boxes, self.pristine)):
            if self.evolve == "shift":
                nx = self.box_nx[i]
                s = k % nx
                sh = lambda a: torch.roll(a.view(*a.shape[:-1], -1, nx), s, dims=-1).reshape(a.shape)  # noqa: E731
                b.T.copy_(sh(T))
                b.Y.copy_(sh(Y))
                b.e.copy_(sh(e))
                b.rho.copy_(sh(self.rho0[i]))
                if b.solid is not None:
                    b.solid.copy_(sh(self.solid0[i]))
                continue
            b.Y.copy_(Y)
            b.rho.copy_(self.rho0[i])               # a shift step may have rolled rho / solid
            if b.solid is not None:
                b.solid.copy_(self.solid0[i])
            if self.evolve != "perturb":
                b.T.copy_(T)
                b.e.copy_(e)
                continue
            g = torch.Generator(device=T.device)
            g.manual_seed(23993 + 7919 * k + 104729 * i)
            u = torch.rand(T.shape, generator=g, device=T.device, dtype=torch.float64)
            Tp = torch.where(self.active[i], (T * (1.0 + self.amp * (2.0 * u - 1.0))).clamp_min(T_MIN), T)
            b.T.copy_(Tp)
            self.chem.energy(b.T, b.Y, out=b.e)

    def step(self, rtol, atol, cost=None):
        import torch
        stats = []
        for c in self.calls:
            bx = [self.boxes[i] for i in c]
            cc = None
            if cost is not None:
                cc = torch.zeros(len(c), dtype=torch.float64, device=self.boxes[0].rho.device)
            stats.append(self.chem.integrate_boxes(bx, rtol=rtol, atol=atol, box_cost=cc))
            if cost is not None:
                cost[c] += cc.cpu().numpy()
        return stats


def _map_species(chem, raw):
    """Expand 9-species H2-air boxes to the ctx's mechanism by species name (NEXT-3 mechanisms)."""
    import torch
    import synth
    src = synth.load_trajectories()["species"]
    dst = chem.mech.species
    if list(dst) == list(src):
        return raw
    for b in raw:
        Y = torch.zeros((len(dst), b["Y"].shape[1]), dtype=b["Y"].dtype, device=b["Y"].device)
        for j, s in enumerate(src):
            Y[dst.index(s)] = b["Y"][j]
        if "NO" in dst:
            no = 1e-4 * Y[dst.index("N2")]
            Y[dst.index("NO")] += no
            Y[dst.index("N2")] -= no
        b["Y"] = Y
    return raw


def _mk_boxes(chem, raw):
    from paper_2510_23993_b200 import Box
    out = []
    raw = _map_species(chem, raw)
    for b in raw:
        e = chem.energy(b["T"], b["Y"])            # e = u(T0, Y) with the CUDA path's own thermo
        out.append(Box(b["rho"], e, b["T"].clone(), b["Y"].clone(), b["dt"], b.get("solid")))
    return out


def _balanced(chem, args, all_ids, build, rank, world, calls_for, home):
    """Cost-weighted box -> rank map: every rank integrates its home boxes once
    (calibration call, box_cost), the per-box costs are all-gathered (NCCL), and the same LPT owner
    map is computed on every rank (sharding.plan); owners regenerate their boxes from the pure
    generator."""
    from paper_2510_23993_b200 import sharding
    mine = home(rank)
    boxes = _mk_boxes(chem, [build(all_ids[i]) for i in mine])
    w0 = Workload(chem, boxes, calls_for(mine), {}, 0, "restore", 0.0)
    cost = np.zeros(len(mine))
    w0.step(args.rtol, args.atol, cost=cost)
    gcost, owner, imb, imb_home = sharding.plan(home, cost, len(all_ids), world, args.balance)
    own = [i for i in range(len(all_ids)) if owner[i] == rank]
    if own == mine:
        boxes = w0.boxes
    else:
        del w0, boxes
        boxes = _mk_boxes(chem, [build(all_ids[i]) for i in own])
    extra = dict(balance=args.balance, imbalance_max_over_mean=imb, imbalance_without_lpt=imb_home,
                 boxes_owned=len(own), calibration="per-box attempted substeps of one call (box_cost)",
                 multi_gpu_status="unmeasured on hardware beyond 1 GPU" if world > 1 else None)
    return own, boxes, extra


def build_workload(args, chem, doc, device, rank, world, config=None, evolve="auto"):
    import synth
    from paper_2510_23993_b200 import mechanism
    # the field generators and the trajectory table speak the 9 H2-air species; boxes are mapped to
    # the ctx's mechanism by name afterwards (_map_species)
    m = chem.mech if chem.mech.name == "h2air_li2004" else mechanism.load("h2air_li2004")
    config = config or args.config
    if evolve == "auto":
        evolve = "restore" if config == "cfg2" else "shift"
    mk = lambda boxes, calls, meta, cs, extra=None: Workload(chem, boxes, calls, meta, cs, evolve,  # noqa: E731
                                                             args.perturb, extra)
    if config == "cfg2":
        raw, meta = synth.field_cfg2(doc, device=device)
        boxes = _mk_boxes(chem, raw)
        return mk(boxes, [list(range(len(boxes)))], meta, sum(b.ncells for b in boxes))
    if config == "cfg2b":
        raw, meta = synth.field_cfg2b(doc, device=device)
        boxes = _mk_boxes(chem, raw)
        return mk(boxes, [list(range(len(boxes)))], meta, sum(b.ncells for b in boxes))
    if config == "cfg3":
        raw, meta = synth.field_cfg3(doc, m.W, m.species, device=device)
        boxes = _mk_boxes(chem, raw)
        return mk(boxes, [list(range(len(boxes)))], meta, sum(b.ncells for b in boxes))
    if config == "cfg5":
        # one field's 128 boxes over the ranks (strong), LPT on a calibration call's box cost
        nb = 128
        ids = list(range(nb))
        _, meta = synth.field_cfg5(doc, m.W, m.species, device=device, box_ids=[])
        build = lambda b: synth.field_cfg5(doc, m.W, m.species, device=device, box_ids=[b])[0][0]  # noqa: E731
        own, boxes, extra = _balanced(chem, args, ids, build, rank, world, lambda idx: [list(range(len(idx)))],
                                      lambda r: list(range(r, nb, world)))
        meta["scaling"] = "strong"
        return mk(boxes, [list(range(len(boxes)))], meta, sum(b.ncells for b in boxes), extra)
    if config == "cfg4":
        # weak scaling: P copies of the 3-level hierarchy; copy p calibrated on rank p, then the
        # P*192 boxes are redistributed by LPT on the measured per-box cost.
        all_desc = [d for p in range(world) for d in synth.hierarchy_cfg4(copy=p)]

        def calls_for(idx):
            lv = [all_desc[i]["level"] for i in idx]
            # one coarse step with subcycling: L0 x1 (dt), L1 x2 (dt/2), L2 x4 (dt/4),
            # fused across levels: {L0,L1,L2}, {L1,L2}, {L2}, {L2}
            return [[k for k, l in enumerate(lv) if l >= 0], [k for k, l in enumerate(lv) if l >= 1],
                    [k for k, l in enumerate(lv) if l >= 2], [k for k, l in enumerate(lv) if l >= 2]]

        own, boxes, extra = _balanced(chem, args, list(range(len(all_desc))),
                                      lambda i: synth.build_cfg4_box(doc, m.W, m.species, all_desc[i], device),
                                      rank, world, calls_for,
                                      lambda r: [i for i, d in enumerate(all_desc) if d["copy"] == r])
        cell_steps = sum(b.ncells * 2 ** all_desc[i]["level"] for b, i in zip(boxes, own))
        meta = dict(workload=f"cfg4: 3-level AMR hierarchy (ratio 2, 32^3 boxes, 192 boxes/copy, 6.3M cells/copy) "
                             f"of detonation fields, {world} copies, subcycled coarse step (4 fused calls), "
                             f"balance={args.balance}", cells=sum(b.ncells for b in boxes))
        return mk(boxes, calls_for(own), meta, cell_steps, extra)
    raise SystemExit(f"unknown --config {config}")


# ------------------------------------------------------------------ timing
def timed(wl, args, steps, warmup, dist=None, before=None, clocks=None, rtol=None, atol=None):
    """warmup + steps steps; each step: prepare(k) (untimed) -> [start event] fused calls (+ the
    §8(e) per-step reductions when N > 1) [end event].  Returns (per-step ms, stats of timed steps)."""
    import torch
    rtol = args.rtol if rtol is None else rtol
    atol = args.atol if atol is None else atol
    for k in range(warmup):
        wl.prepare(k)
        if before:
            before()
        wl.step(rtol, atol)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    stats, reds = [], []
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    if clocks:
        clocks.start()
    wall = []
    for k in range(steps):
        wl.prepare(warmup + k)
        if before:
            before()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev[k][0].record()
        st = wl.step(rtol, atol)
        if dist is not None:
            reds.append(step_reductions(st, wl))
        ev[k][1].record()
        ev[k][1].synchronize()
        wall.append((time.perf_counter() - t0) * 1e3)   # host wall clock around the step
        stats += st
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clk = clocks.stop() if clocks else None
    timed.last_wall_ms = wall
    return [a.elapsed_time(b) for a, b in ev], stats, clk, reds


def step_reductions(stats, wl):
    """SURVEY §8(e) (2)-(3) every step: SUM of unfinished cells and attempted substeps (convergence),
    MIN of the proposed next dt (the CFL stand-in: halve it if any cell ran out of budget)."""
    from paper_2510_23993_b200 import sharding
    unf = sum(s["n_unfinished"] for s in stats)
    att = sum(s["steps_attempted"] for s in stats)
    return sharding.step_reductions(unf, att, min(b.dt for b in wl.boxes) * (0.5 if unf else 1.0))


def roofline(fm, stats, peak_derived, peak_measured):
    flops = sum(fm.flops(s) for s in stats)
    k_ms = sum(s["t_bulk_ms"] + s["t_sparse_ms"] for s in stats)
    ach = flops / (k_ms / 1e3) / 1e12 if k_ms > 0 else 0.0
    return flops, k_ms, ach


# ------------------------------------------------------------------ oracle (cpu baseline / reference arm)
def host_info():
    model, smt = None, None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        smt = open("/sys/devices/system/cpu/smt/active").read().strip() == "1"
    except OSError:
        pass
    return dict(cpu_model=model or platform.processor(), smt=smt, nproc=os.cpu_count())


def host_threads(o):
    """Threads for the oracle baseline: every host core this process may run on.  torchrun exports
    OMP_NUM_THREADS=1 to its ranks, which would time the reference arm / cpu_baseline on one core."""
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count() or 1
    return max(n, o.max_threads())


def oracle_sample(meta, seconds_target, rtol, atol):
    """Time the oracle, as it stands, on a bounded sample of the workload's cells (all host cores)."""
    from oracle import Oracle
    o = Oracle("h2air_li2004")
    st = meta["state"]
    Y = np.asarray(st["Y"])
    e = o.energy(st["T"], Y)
    nth = host_threads(o)

    def run(n, threads=nth):
        t0 = time.perf_counter()
        o.integrate_cells(np.full(n, st["rho"]), np.full(n, e), np.full(n, st["T"]), np.tile(Y, (n, 1)), 1e-7,
                          rtol=rtol, atolY=atol, atolT=ATOL_T, nthreads=threads)
        return time.perf_counter() - t0

    n = nth
    dt = run(n)
    while dt < 0.5 and n < 1 << 22:         # calibrate the sample to ~seconds_target of CPU work
        n *= 4
        dt = run(n)
    n = int(max(nth, min(1 << 24, n * seconds_target / max(dt, 1e-9))))
    dt = run(n)
    n1 = max(1, int(n / nth / 4))
    dt1 = run(n1, 1)
    return dict(cells=n, seconds=dt, threads=nth, value=n / dt / 1e6, one_core_value=n1 / dt1 / 1e6)


def _meta_cfg2(doc):
    import synth
    tr = next(t for t in doc["trajectories"] if t["kind"] == "fresh" and t["T0"] == 1200.0)
    rho, T, Y = synth.traj_state(tr, 0.9)
    return dict(workload="cfg2: uniform 128^3 H2-air field, T0=1200 K traj. state at t=0.9 tau, 64 boxes of 32^3, "
                         "dt=1e-07 s", cells=128 ** 3, state=dict(rho=float(rho), T=float(T), Y=np.asarray(Y).tolist()))


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
                                       "(all cells of cfg2 are identical)", **host_info()},
            "e2e": {"value": value, "unit": "Mcell-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def oracle_stratified(chem, wl, rtol, atol, seconds_target, n_prop=65536, n_heavy=1000):
    """cpu_baseline for a non-uniform field (SURVEY §8(d) / BASELINE.md §3): the cells of this rank's
    field are split into classes by the substeps the GPU needed for them in one (untimed) call of the
    first fused call of a step: cold/gated (no work on either side), log2 substep bins, and the
    n_heavy heaviest cells as a class of their own.  A proportional sample of >= n_prop cells plus
    all heavy cells is integrated by the oracle (as it stands, same rtol/atol as the GPU) on all host
    cores, class by class; the field time is extrapolated as sum_class (class time / sampled cells x
    class count) and LABELLED an extrapolation.  A sub-sample is also timed on one core."""
    import torch
    from oracle import Oracle
    o = Oracle(chem.mech.name)
    wl.prepare(0)
    # pristine inputs (the named config), one GPU call for the per-cell substep counts
    for b, (T, Y, e) in zip(wl.boxes, wl.pristine):
        b.T.copy_(T); b.Y.copy_(Y); b.e.copy_(e)
    first = wl.calls[0]
    chem.integrate_boxes([wl.boxes[i] for i in first], rtol=rtol, atol=atol)
    _, steps = chem.cell_status(substeps=True)
    steps = steps.cpu().numpy().astype(np.int64)
    sizes = [wl.boxes[i].ncells for i in first]
    starts = np.cumsum([0] + sizes)
    active = steps > 0
    ids = np.nonzero(active)[0]
    heavy = ids[np.argsort(steps[ids], kind="stable")[::-1][:n_heavy]]
    rest = np.setdiff1d(ids, heavy)
    bins = np.floor(np.log2(np.maximum(steps[rest], 1))).astype(int)
    rng = np.random.default_rng(23993)
    frac = min(1.0, n_prop / max(len(rest), 1))
    classes = [("heavy_top%d" % n_heavy, heavy, heavy)]
    for bv in np.unique(bins):
        pool = rest[bins == bv]
        k = min(len(pool), max(64, int(round(frac * len(pool)))))
        classes.append((f"substeps_2^{bv}", pool, np.sort(rng.choice(pool, size=k, replace=False))))

    def gather(sel):
        bidx = np.searchsorted(starts, sel, side="right") - 1
        rho, T, Y, e, dt = [], [], [], [], []
        for bi in np.unique(bidx):
            offs = torch.as_tensor(sel[bidx == bi] - starts[bi], device=wl.boxes[0].rho.device)
            b = wl.boxes[first[bi]]
            T0, Y0, _ = wl.pristine[first[bi]]
            rho.append(b.rho[offs].cpu().numpy()); T.append(T0[offs].cpu().numpy())
            Y.append(Y0[:, offs].cpu().numpy().T); dt += [b.dt] * len(offs)
        rho, T, Y, dt = np.concatenate(rho), np.concatenate(T), np.concatenate(Y), np.array(dt)
        e = np.array([o.energy(t, y) for t, y in zip(T, Y)])    # the oracle's own thermo
        return rho, e, T, Y, dt

    nth = host_threads(o)

    def run(data, threads):
        rho, e, T, Y, dt = data
        t0 = time.perf_counter()
        for d in np.unique(dt):
            s = dt == d
            o.integrate_cells(rho[s], e[s], T[s], Y[s], float(d), rtol=rtol, atolY=atol, atolT=ATOL_T,
                              nthreads=threads)
        return time.perf_counter() - t0

    field_s, one_core_s, sampled, per_class = 0.0, 0.0, 0, {}
    for name, pool, sel in classes:
        data = gather(sel)
        t = run(data, nth)
        field_s += t * len(pool) / len(sel)
        sub = max(1, len(sel) // 64)
        t1 = run(tuple(x[:sub] for x in data), 1)
        one_core_s += t1 * len(pool) / sub
        sampled += len(sel)
        per_class[name] = dict(count=int(len(pool)), sampled=int(len(sel)), seconds=round(t, 3),
                               mean_gpu_substeps=float(steps[pool].mean()))
    total_cells = int(sum(sizes))
    return dict(value=total_cells / field_s / 1e6, one_core_value=total_cells / one_core_s / 1e6, threads=nth,
                classes=per_class,
                sample=(f"stratified: {sampled} of {len(ids)} active cells ({len(classes) - 1} GPU-substep classes "
                        f"proportional, >= 64 each, plus the {len(heavy)} heaviest), oracle at the GPU's rtol/atol on "
                        f"{nth} threads, extrapolated per class to the {total_cells}-cell field of one fused call "
                        f"(gated cells cost 0)"))


# ------------------------------------------------------------------ our arm
def measure(args, chem, doc, device, rank, world, dist, config, fm, peaks, with_variants, clocks=None):
    """Build `config`, time the default schedule (headline), then optionally Alg. 3, the first call
    of a layout and exact replay.  Returns (workload, result dict)."""
    import torch
    wl = build_workload(args, chem, doc, device, rank, world, config=config, evolve=args.evolve)
    steps_ms, stats, clk, reds = timed(wl, args, args.steps, args.warmup, dist, clocks=clocks)
    wall_ms = float(np.median(timed.last_wall_ms))
    t_rank = sum(steps_ms) / 1e3
    t_total, tot_cs = t_rank, float(wl.cell_steps)
    if world > 1:
        from paper_2510_23993_b200 import sharding
        t_total = float(sharding.reduce_stats([t_rank], "max")[0])          # max over ranks
        tot_cs = float(sharding.reduce_stats([float(wl.cell_steps)], "sum")[0])
    flops, k_ms, ach = roofline(fm, stats, *peaks)
    res = dict(value=tot_cs * args.steps / t_total / 1e6, ms_per_step=1e3 * t_total / args.steps,
               steps_ms=steps_ms, t_rank=t_rank, stats=stats, flops=flops, k_ms=k_ms, achieved=ach,
               clocks=clk, reductions=reds[-1] if reds else None, tot_cs=tot_cs, wall_ms=wall_ms)
    if with_variants and config != "cfg2" and not args.no_schedules:
        var = {}
        chem_opts0 = dict(schedule_lpt=chem.opts.schedule_lpt)

        def forget():
            chem.forget_hints()

        for name, kw in (("first_call_no_hints", dict(before=forget)),
                         ("alg3_schedule_lpt0", dict(opt=dict(schedule_lpt=0))),
                         ("replayed_exact_hints", dict(evolve="restore"))):
            if "opt" in kw:
                chem.set_opts(**kw["opt"])
            ev0 = wl.evolve
            if "evolve" in kw:
                wl.evolve = kw["evolve"]
            n = max(3, min(args.steps, 10))
            ms, st, _, _ = timed(wl, args, n, 2, dist, before=kw.get("before"))
            wl.evolve = ev0
            chem.set_opts(**chem_opts0)
            t = sum(ms) / 1e3
            if world > 1:
                from paper_2510_23993_b200 import sharding
                t = float(sharding.reduce_stats([t], "max")[0])
            fl, km, a = roofline(fm, st, *peaks)
            s0 = st[-1]
            var[name] = dict(value=tot_cs * n / t / 1e6, ms_per_step=1e3 * t / n, steps=n,
                             frac=a / peaks[0], lpt=s0.get("lpt", 0), lockstep=s0["lockstep"],
                             bulk_iters=s0["bulk_iters"], sparse_cells=s0["sparse_cells"],
                             t_sparse_ms=s0["t_sparse_ms"], hint_accuracy=s0.get("hint_accuracy"))
        res["schedules"] = var
    if with_variants and not args.no_prod:
        # SURVEY §8(d) secondary number: production tolerance (rtol 1e-6, atol_Y 1e-12, atol_T 1e-3 K)
        chem.set_opts(atol_T=PROD_TOL["atol_T"])
        n = max(3, min(args.steps, 10))
        ms, st, _, _ = timed(wl, args, n, 2, dist, rtol=PROD_TOL["rtol"], atol=PROD_TOL["atol"])
        chem.set_opts(atol_T=ATOL_T)
        t = sum(ms) / 1e3
        if world > 1:
            from paper_2510_23993_b200 import sharding
            t = float(sharding.reduce_stats([t], "max")[0])
        fl, km, a = roofline(fm, st, *peaks)
        res["production_tolerance"] = dict(value=tot_cs * n / t / 1e6, ms_per_step=1e3 * t / n, frac=a / peaks[0],
                                           substeps_per_cell_step=sum(s["steps_attempted"] for s in st) / n
                                           / max(wl.cell_steps, 1),
                                           tolerances=PROD_TOL)
    torch.cuda.synchronize()
    return wl, res


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
    pg = dist if world > 1 else None
    method = METHODS[args.method]
    chem = Chem(args.mech, device=local, atol_T=ATOL_T, method=method, **_opts(args))
    doc = synth.load_trajectories()
    fm = FlopModel(chem.mech, stages=STAGES[method])
    sm_mhz_peak = 1965.0
    try:
        sm_mhz_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("sm_max_mhz", sm_mhz_peak))
    except Exception:
        pass
    peak = fp64_peak_tflops(sm_mhz=sm_mhz_peak)
    peak_meas = None
    try:
        peak_meas = float(json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))["tflops"])
    except Exception:
        pass

    clocks = ClockSampler(local)
    wl, res = measure(args, chem, doc, device, rank, world, pg, args.config, fm, (peak, peak_meas), True,
                      clocks=clocks)
    stats = res["stats"]
    ncells = wl.ncells

    traffic, ncu_pipe = None, None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(args.config)
        if tr:
            traffic, ncu_pipe = tr["traffic_bytes_per_launch"], tr.get("ncu_fp64_pipe_pct")
    except Exception:
        pass

    # e2e through the public API with host buffers (H2D + calls + D2H inside the timed region); the
    # host inputs alternate between two perturbed realisations when the device run perturbs
    e2e = None
    if not args.no_e2e:
        def host_set(k):
            wl.prepare(k)
            return [dict(rho=b.rho.cpu().pin_memory(), e=b.e.cpu().pin_memory(), T=b.T.cpu().pin_memory(),
                         Y=b.Y.cpu().pin_memory(), dt=b.dt) for b in wl.boxes]
        sets = [host_set(1000)] + ([host_set(1001)] if wl.evolve != "restore" else [])
        # copy/compute pipelining groups: dense fields split into ~0.25 GB groups (3..12; measured r02:
        # cfg2 3 groups 147 vs 5 groups 144, cfg5 12 groups 181 vs 5 groups 167 Mcell-steps/s); the
        # detonation fields run as one call (splitting them splits the heavy-first schedule)
        field_bytes = sum(b.ncells * (3 + b.Y.shape[0]) * 8 for b in wl.boxes)
        chunks = args.e2e_chunks if args.e2e_chunks > 0 else \
            (int(min(12, max(3, round(field_bytes / 0.25e9)))) if args.config in ("cfg2", "cfg2b", "cfg5") else 1)
        hr = HostRunner(chem, sets[0], wl.calls, chunks=chunks, taper=args.e2e_taper)
        for k in range(2):
            hr.load_inputs(sets[k % len(sets)])
            hr.step(args.rtol, args.atol)
        torch.cuda.synchronize()
        e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(args.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        d2h_steps, h2d_steps = [], []
        for k in range(args.steps):
            hr.load_inputs(sets[k % len(sets)])       # host memcpy into the pinned slab, untimed
            e_ev[k][0].record()
            hr.step(args.rtol, args.atol)
            e_ev[k][1].record()
            d2h_steps.append(hr.d2h_bytes)
            h2d_steps.append(hr.h2d_bytes)
        torch.cuda.synchronize()
        te = sum(a.elapsed_time(b) for a, b in e_ev) / 1e3
        if world > 1:
            from paper_2510_23993_b200 import sharding
            te = float(sharding.reduce_stats([te], "max")[0])
        e2e = {"value": res["tot_cs"] * args.steps / te / 1e6, "unit": "Mcell-steps/s",
               "h2d_bytes_per_step": float(np.mean(h2d_steps)), "d2h_bytes_per_step": float(np.mean(d2h_steps)),
               "copy_note": "H2D: every box's T, then rho/e/Y of boxes with active cells (chem_box_active) on the "
                            "unpipelined path, the whole slab on the pipelined one; D2H: T, Y of the boxes the step "
                            f"touched (box_cost > 0) (full field: {hr.h2d_bytes_full} B in, {hr.d2h_bytes_full} B out)",
               "copy_compute_chunks": chunks if hr.pipelined else 1,
               "taper": args.e2e_taper if hr.pipelined else None,
               "inputs": f"two alternating {wl.evolve}ed host sets" if len(sets) > 1 else "pristine host inputs"}
        del hr, sets

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if args.config == "cfg2" and args.mech == "h2air_li2004":
            r = oracle_sample(wl.meta, args.cpu_sample_seconds, args.rtol, args.atol)
            cpu = {"value": r["value"], "unit": "Mcell-steps/s", "cores": r["threads"], "kind": "oracle",
                   "one_core_value": r["one_core_value"],
                   "sample": f"{r['cells']} cells of the cfg2 state (all cfg2 cells are identical), "
                             f"{r['seconds']:.1f} s on {r['threads']} threads, same rtol/atol as the GPU run",
                   **host_info()}
        else:
            r = oracle_stratified(chem, wl, args.rtol, args.atol, args.cpu_sample_seconds)
            cpu = {"value": r["value"], "unit": "Mcell-steps/s", "cores": r["threads"], "kind": "oracle",
                   "one_core_value": r["one_core_value"], "sample": r["sample"], "extrapolated": True,
                   "classes": r["classes"], **host_info()}

    # extra configs timed into the same line (the driver runs only the default command)
    also = []
    also_cfgs = (["cfg2b", "cfg3"] if args.config == "cfg2" else []) if args.also == "auto" else \
        [c for c in args.also.split(",") if c and c != "none"]
    if world == 1 and also_cfgs:
        meta_main, wl_cells, wl_cs, wl_calls, wl_extra = wl.meta, ncells, wl.cell_steps, len(wl.calls), wl.extra
        n_boxes, wl_evolve = len(wl.boxes), wl.evolve
        del wl
        chem.release_workspaces()
        torch.cuda.empty_cache()
        for c in also_cfgs:
            a = argparse.Namespace(**{**vars(args), "no_prod": True})
            w2, r2 = measure(a, chem, doc, device, rank, world, pg, c, fm, (peak, peak_meas), True)
            s0 = r2["stats"][-1]
            also.append(dict(config=c, workload=w2.meta["workload"], schedule="default (heavy-first when the "
                             "previous step's hints are skewed)", inputs=w2.evolve, value=r2["value"],
                             ms_per_step=r2["ms_per_step"], frac=r2["achieved"] / peak, lpt=s0.get("lpt", 0),
                             hint_accuracy=s0.get("hint_accuracy"),
                             sparse_cells=s0["sparse_cells"], bulk_iters=s0["bulk_iters"],
                             substeps_per_cell_step=sum(s["steps_attempted"] for s in r2["stats"]) / args.steps
                             / max(w2.cell_steps, 1), schedules=r2.get("schedules")))
            del w2
            chem.release_workspaces()
            torch.cuda.empty_cache()
    else:
        meta_main, wl_cells, wl_cs, wl_calls, wl_extra = wl.meta, ncells, wl.cell_steps, len(wl.calls), wl.extra
        n_boxes, wl_evolve = len(wl.boxes), wl.evolve

    att = sum(s["steps_attempted"] for s in stats) / args.steps
    acc = sum(s["steps_accepted"] for s in stats) / args.steps
    s0 = stats[-1]
    launches_int = sum(s["bulk_iters"] + (1 if s["sparse_cells"] > 0 else 0) for s in stats)
    gpu_launches = sum(s["kernel_launches"] for s in stats)   # the library's own count (chem_stats)
    if rank == 0:
        line = {
            "metric": METRIC, "value": res["value"], "unit": "Mcell-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
            "scaling": meta_main.get("scaling", "weak"), "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": meta_main["workload"] + ("" if args.mech == "h2air_li2004" else
                                                            f" [mechanism {args.mech}, {chem.ns} species]"),
                       "mechanism": args.mech, "cells_per_gpu": wl_cells, "boxes_per_gpu": n_boxes,
                       "cell_steps_per_step_per_gpu": wl_cs, "fused_calls_per_step": wl_calls,
                       "rtol": args.rtol, "atol_Y": args.atol, "atol_T": ATOL_T, "method": args.method,
                       **({"opts": args.opt} if args.opt else {}),
                       "inputs_between_steps": {"restore": "restored (cfg2: every cell the same state)",
                                                "shift": "field rolled one cell along x per step inside every "
                                                         "box (front advancing; cost hints one cell stale)",
                                                "perturb": f"seeded +-{args.perturb:g} T jitter per step, e "
                                                           "recomputed"}[wl_evolve],
                       "l2": "inputs >= 369 MB/GPU > 126 MB L2 (no flush needed)",
                       "parallelism": f"boxes over {world} rank(s)",
                       "schedule": "heavy-first (cost hints: the previous step's per-cell substeps)"
                                   if s0.get("lpt", 0) else "bulk-sparse (Alg. 3)",
                       **wl_extra},
            "roofline": {"bound": "alu", "achieved": res["achieved"], "peak": peak, "unit": "TFLOP/s",
                         "frac": res["achieved"] / peak, "traffic": traffic, "traffic_unit": "bytes per launch (ncu)",
                         "peak_measured_dfma": peak_meas,
                         "frac_vs_measured_dfma": (res["achieved"] / peak_meas) if peak_meas else None,
                         "ncu_fp64_pipe_pct": ncu_pipe, "kernel": "k_integrate (bulk+sparse launches)",
                         "flops_model": fm.table(), "flops_timed": res["flops"],
                         "k_integrate_ms_timed": res["k_ms"],
                         "peak_source": "148 SMs x 64 FP64 FMA/clk x 2 x sm_max_mhz (derived, DESIGN.md §5); "
                                        "measured DFMA loop: profiles/fp64_peak.json"},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": gpu_launches, "clocks": res["clocks"],
            "schedules": res.get("schedules"), "production_tolerance": res.get("production_tolerance"),
            "also": also or None,
            "detail": {"step_ms": res["steps_ms"], "step_ms_median": float(np.median(res["steps_ms"])),
                       "step_ms_min": float(np.min(res["steps_ms"])), "step_ms_max": float(np.max(res["steps_ms"])),
                       "host_wall_ms_per_step": res.get("wall_ms"), "rank0_seconds": res["t_rank"],
                       "k_integrate_ms": res["k_ms"] / args.steps,
                       "integrate_launches": launches_int, "substeps_per_cell_step": att / max(wl_cs, 1),
                       "accepted_per_cell_step": acc / max(wl_cs, 1),
                       # SURVEY §8(d) "also reported" rates, this rank's calls over the (max-over-ranks) step time
                       "rates_per_s": {k: sum(s[f] for s in stats) / (res["ms_per_step"] * args.steps * 1e-3)
                                       for k, f in (("active_cell_steps", "active0"),
                                                    ("substeps_attempted", "steps_attempted"),
                                                    ("rhs_evals", "rhs_evals"))},
                       "frozen_per_cell_step": sum(s.get("steps_frozen", 0) for s in stats) / args.steps
                       / max(wl_cs, 1), "bulk_iters": s0["bulk_iters"],
                       "active_per_iter": s0["active_per_iter"], "sparse_cells": s0["sparse_cells"],
                       "active0": s0["active0"], "t_gate_ms": s0["t_gate_ms"], "t_compact_ms": s0["t_compact_ms"],
                       "t_sparse_ms": s0["t_sparse_ms"], "n_unfinished": s0["n_unfinished"],
                       "n_nonfinite": s0["n_nonfinite"], "max_energy_drift": s0["max_energy_drift"],
                       "lockstep": s0["lockstep"], "lpt": s0.get("lpt", 0),
                       "hint_accuracy": s0.get("hint_accuracy"),
                       "bulk_simt_eff": s0["bulk_substeps"] / max(32 * s0["warp_substeps"], 1),
                       "step_reductions": res["reductions"]},
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

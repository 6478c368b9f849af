"""NEXT-2: re-derive the paper's schedule constants on B200 (PAPER.md P:179 K_max = 5 "from timing
experiments", P:181 N*_active = 1e4 "manually tuned", App. D saturation, App. E fusion).

    python tools/sweep_schedule.py [cfg3 cfg4 ...]     (on a GPU box; prints JSON lines)

For each config: time one step (the bench's fused calls) for K_max_bulk x N* (and the paper's
all-cells bulk mode), plus the fusion experiment: the same cells as 1..N boxes in one fused call vs
one call per box.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2510_23993_b200 import Box, Chem  # noqa: E402


def time_step(wl, chem, reps=3):
    """Median of `reps` steps after one warm-up step, inputs as the bench prepares them (shifted field)."""
    ts = []
    for k in range(reps + 1):
        wl.prepare(k)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        st = wl.step(bench.RTOL, bench.ATOL)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts[1:])), st


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["cfg3", "cfg4"])
    ap.add_argument("--kmax", default="5,20,100")
    ap.add_argument("--nstar", default="1e4,3e4,1e5,3e5,1e9")
    ap.add_argument("--lpt", default="0", help="schedule_lpt values to sweep (0 = Alg. 3, 2 = auto heavy-first)")
    ap.add_argument("--no-fusion", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    doc = synth.load_trajectories()
    chem = Chem("h2air_li2004", device=0, atol_T=bench.ATOL_T)
    for cfg in args.configs:
        a = argparse.Namespace(config=cfg, rtol=bench.RTOL, atol=bench.ATOL, balance="none", perturb=0.01,
                               evolve="auto")
        wl = bench.build_workload(a, chem, doc, dev, 0, 1, config=cfg, evolve="auto")
        base = None
        for lp in [int(x) for x in args.lpt.split(",")]:
          for km in [int(x) for x in args.kmax.split(",")]:
            for ns in [int(float(x)) for x in args.nstar.split(",")]:
                chem.set_opts(kmax_bulk=km, n_active_star=ns, compact_bulk=1, schedule_lpt=lp)
                ms, st = time_step(wl, chem)
                base = base or ms
                print(json.dumps(dict(exp="schedule", config=cfg, kmax_bulk=km, n_active_star=ns, compact_bulk=1,
                                      schedule_lpt=lp,
                                      ms_per_step=ms, bulk_iters=sum(s["bulk_iters"] for s in st),
                                      sparse_cells=sum(s["sparse_cells"] for s in st),
                                      Mcell_steps_per_s=wl.cell_steps / ms / 1e3)), flush=True)
        if args.no_fusion:
            continue
        chem.set_opts(kmax_bulk=5, n_active_star=10000, compact_bulk=0, schedule_lpt=0)   # Alg. 3 as written
        ms, st = time_step(wl, chem)
        print(json.dumps(dict(exp="schedule", config=cfg, kmax_bulk=5, n_active_star=10000, compact_bulk=0,
                              ms_per_step=ms, bulk_iters=sum(s["bulk_iters"] for s in st),
                              Mcell_steps_per_s=wl.cell_steps / ms / 1e3, note="paper: bulk over all cells")),
              flush=True)
        chem.set_opts(kmax_bulk=5, n_active_star=-1, compact_bulk=1, schedule_lpt=2)
        del wl
        torch.cuda.empty_cache()
    if args.no_fusion:
        return
    # App. E fusion experiment: 1M cells of cfg2 state split into 1..512 boxes, one fused call vs a call per box
    raw, _ = synth.field_cfg2(doc, side=128, box=32, device=dev)
    st0 = raw[0]
    total = 1 << 20
    for nb in (1, 8, 64, 512):
        nc = total // nb
        boxes = []
        for _ in range(nb):
            T = st0["T"][:1].expand(nc).clone()
            Y = st0["Y"][:, :1].expand(-1, nc).contiguous()
            rho = st0["rho"][:1].expand(nc).clone()
            boxes.append(Box(rho, chem.energy(T, Y), T, Y, 1e-7))
        pr = [(b.T.clone(), b.Y.clone()) for b in boxes]

        def run(fused):
            for b, (T, Y) in zip(boxes, pr):
                b.T.copy_(T); b.Y.copy_(Y)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if fused:
                chem.integrate_boxes(boxes, rtol=bench.RTOL, atol=bench.ATOL)
            else:
                for b in boxes:
                    chem.integrate_boxes([b], rtol=bench.RTOL, atol=bench.ATOL)
            torch.cuda.synchronize()
            return (time.perf_counter() - t0) * 1e3

        run(True); run(False)
        f = min(run(True) for _ in range(2))
        u = min(run(False) for _ in range(2))
        print(json.dumps(dict(exp="fusion", cells=total, boxes=nb, fused_ms=f, per_box_ms=u, speedup=u / f)), flush=True)


if __name__ == "__main__":
    main()

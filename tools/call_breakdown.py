"""Per-call breakdown of one bench step (the fused chem_integrate_boxes calls of a config): cells, active
cells, attempted substeps, schedule, phase times, and each call's FP64 fraction by the §8(d) model — shows
which calls of a multi-call step (cfg4's subcycled AMR levels) run below the whole-step rate.

    python tools/call_breakdown.py --config cfg4
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import synth
    from paper_2510_23993_b200 import Chem
    from paper_2510_23993_b200.flops import FlopModel, fp64_peak_tflops

    args = bench.parse()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    method = bench.METHODS[args.method]
    chem = Chem(args.mech, device=0, atol_T=bench.ATOL_T, method=method, **bench._opts(args))
    wl = bench.build_workload(args, chem, synth.load_trajectories(), dev, 0, 1, config=args.config, evolve=args.evolve)
    fm = FlopModel(chem.mech, stages=bench.STAGES[method])
    peak = fp64_peak_tflops(sm_mhz=1965.0)
    for k in range(3):
        wl.prepare(k)
        wl.step(args.rtol, args.atol)
    wl.prepare(3)
    torch.cuda.synchronize()
    rows = []
    for c in wl.calls:
        bx = [wl.boxes[i] for i in c]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st = chem.integrate_boxes(bx, rtol=args.rtol, atol=args.atol)
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b)
        fl = fm.flops(st) if hasattr(fm, "flops") else None
        kern = st["t_bulk_ms"] + st["t_sparse_ms"]
        rows.append(dict(boxes=len(c), cells=st["cells"], active0=st["active0"], attempted=st["steps_attempted"],
                         lpt=st["lpt"], lockstep=st["lockstep"], bulk_iters=st["bulk_iters"],
                         sparse=st["sparse_cells"], call_ms=round(ms, 3), bulk_ms=round(st["t_bulk_ms"], 3),
                         sparse_ms=round(st["t_sparse_ms"], 3), gate_ms=round(st["t_gate_ms"], 3),
                         substeps_per_ms=round(st["steps_attempted"] / max(kern, 1e-9), 1),
                         frac=(round(fl / (kern * 1e-3) / (peak * 1e12), 3) if fl else None)))
    for r in rows:
        print(json.dumps(r))


if __name__ == "__main__":
    main()

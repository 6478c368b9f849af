"""Per-call breakdown of one bench step (GPU): for each fused call of the step, cells, active cells,
schedule, phase times and substeps.

    python tools/call_probe.py cfg4
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2510_23993_b200 import Chem  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    doc = synth.load_trajectories()
    dev = torch.device("cuda", 0)
    chem = Chem("h2air_li2004", device=0, atol_T=bench.ATOL_T)
    a = argparse.Namespace(config=cfg, rtol=bench.RTOL, atol=bench.ATOL, balance="none", perturb=0.01, evolve="auto")
    wl = bench.build_workload(a, chem, doc, dev, 0, 1, config=cfg)
    for k in range(3):
        wl.prepare(k)
        torch.cuda.synchronize()
        for ci, c in enumerate(wl.calls):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            st = chem.integrate_boxes([wl.boxes[i] for i in c], rtol=bench.RTOL, atol=bench.ATOL)
            e.record()
            torch.cuda.synchronize()
            if k == 2:
                print(json.dumps(dict(call=ci, boxes=len(c), cells=st["cells"], active0=st["active0"],
                                      bulk_iters=st["bulk_iters"], sparse=st["sparse_cells"], lpt=st["lpt"],
                                      ms=round(s.elapsed_time(e), 2), t_bulk=round(st["t_bulk_ms"], 2),
                                      t_sparse=round(st["t_sparse_ms"], 2),
                                      substeps=st["steps_attempted"])), flush=True)


if __name__ == "__main__":
    main()

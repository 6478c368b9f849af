"""Bulk SIMT efficiency (lane substeps / (32 x warp substeps)) and step time per bench config, with
lockstep off and on (chem_opts.lockstep; the auto mode's input).

    python tools/simt_stats.py [cfg2 cfg3 ...]        (on a GPU box)
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2510_23993_b200 import Chem  # noqa: E402


def main():
    cfgs = sys.argv[1:] or ["cfg2", "cfg3", "cfg4", "cfg5"]
    doc = synth.load_trajectories()
    dev = torch.device("cuda", 0)
    for cfg in cfgs:
        chem = Chem("h2air_li2004", device=0, atol_T=bench.ATOL_T)
        a = argparse.Namespace(config=cfg, rtol=bench.RTOL, atol=bench.ATOL, balance="none", perturb=0.01,
                               evolve="auto")
        wl = bench.build_workload(a, chem, doc, dev, 0, 1, config=cfg)
        for lock in (0, 1, 2, 2):
            chem.set_opts(lockstep=lock)
            wl.prepare(0)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            st = wl.step(bench.RTOL, bench.ATOL)
            e.record()
            torch.cuda.synchronize()
            ws = sum(x["warp_substeps"] for x in st)
            ls = sum(x["bulk_substeps"] for x in st)
            print(cfg, "lockstep", lock, "used", [x["lockstep"] for x in st][:4], "ms", round(s.elapsed_time(e), 2),
                  "simt_eff(all bulk)", round(ls / max(32 * ws, 1), 3), "frozen", sum(x["steps_frozen"] for x in st),
                  flush=True)
        del wl, chem
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

"""App. B activity trace of one cfg4 coarse step (3 AMR levels) in the paper's line format.

    python tools/activity_trace.py > profiles/r01_activity_trace_cfg4.txt
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2510_23993_b200 import Box, Chem, load_mechanism  # noqa: E402
from paper_2510_23993_b200.api import activity_lines  # noqa: E402

dev = torch.device("cuda", 0)
m = load_mechanism("h2air_li2004")
doc = synth.load_trajectories()
descs = synth.hierarchy_cfg4(copy=0)
raw = [synth.build_cfg4_box(doc, m.W, m.species, d, dev) for d in descs]
chem = Chem("h2air_li2004", device=0, atol_T=1e-6)
boxes = [Box(b["rho"], chem.energy(b["T"], b["Y"]), b["T"].clone(), b["Y"].clone(), b["dt"]) for b in raw]
tr = chem.set_trace(64, len(boxes))
st = chem.integrate_boxes(boxes, rtol=1e-9, atol=1e-20)
rows = min(64, st["bulk_iters"] + 1)
for line in activity_lines(tr[:rows], boxes, levels=[d["level"] for d in descs], t=0.0, kmax=5):
    if not line.endswith("n_active = 0") or ", step = 0," in line:
        print(line)

"""Tail probe (GPU): per-cell attempted substeps of one fused cfg3 call, read from the workspace
(cell_steps), to relate the sparse phase's duration to the heaviest cells' substep counts.

    python tools/tail_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2510_23993_b200 import Box, Chem, load_mechanism  # noqa: E402

m = load_mechanism("h2air_li2004")
doc = synth.load_trajectories()
chem = Chem("h2air_li2004", device=0, atol_T=1e-6)
raw, _ = synth.field_cfg3(doc, m.W, m.species, device=torch.device("cuda", 0))
boxes = []
for b in raw:
    e = chem.energy(b["T"], b["Y"])
    boxes.append(Box(b["rho"], e, b["T"].clone(), b["Y"].clone(), b["dt"], b.get("solid")))
for rep in range(2):
    for bx, b in zip(boxes, raw):
        bx.T.copy_(b["T"]); bx.Y.copy_(b["Y"])
    st = chem.integrate_boxes(boxes)
torch.cuda.synchronize()
N, B = sum(b.ncells for b in boxes), len(boxes)
al = lambda x: (x + 255) & ~255
o = al(15 * 8); o = al(o + B * 56); o = al(o + (B + 1) * 8)    # stats, boxes, box prefix
o = al(o + 8 * N); o = al(o + 8 * N)                            # cell_t, cell_h
steps = chem._ws[o:o + 4 * N].view(torch.int32).cpu().numpy()
st_o = al(al(o + 4 * N) + 4 * N)                                # cell_box, then state
state = chem._ws[st_o:st_o + N].cpu().numpy() & 0x7f
act = steps[state != 0]
q = np.percentile(act, [50, 90, 99, 99.9, 100])
print(f"active {len(act)}  substeps p50/p90/p99/p99.9/max = {q}")
print(f"bulk iters {st['bulk_iters']}, sparse cells {st['sparse_cells']}, t_bulk {st['t_bulk_ms']:.1f} ms, "
      f"t_sparse {st['t_sparse_ms']:.1f} ms")
srt = np.sort(act)[::-1]
for k in (1, 10, 100, 1000, 10000, 36000):
    if k <= len(srt):
        print(f"  {k}-th heaviest cell: {srt[k - 1]} substeps")

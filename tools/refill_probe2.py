"""Bulk vs sparse-only (lane refill) on heterogeneous cells: 8 boxes of the cfg5 field."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_2510_23993_b200 import Box, Chem, load_mechanism
dev = torch.device("cuda", 0)
m = load_mechanism("h2air_li2004")
doc = synth.load_trajectories()
raw, _ = synth.field_cfg5(doc, m.W, m.species, device=dev, box_ids=[1, 2, 9, 10, 17, 18, 25, 26])
chem = Chem("h2air_li2004", device=0, atol_T=1e-6)
boxes = [Box(b["rho"], chem.energy(b["T"], b["Y"]), b["T"].clone(), b["Y"].clone(), b["dt"]) for b in raw]
pr = [(b.T.clone(), b.Y.clone()) for b in boxes]
mode = sys.argv[1] if len(sys.argv) > 1 else "both"
for ns, label in ((10**4, "bulk"), (10**9, "sparse-only")):
    if mode != "both" and mode != label:
        continue
    chem.set_opts(n_active_star=ns)
    for rep in range(2):
        for b, (T, Y) in zip(boxes, pr):
            b.T.copy_(T); b.Y.copy_(Y)
        torch.cuda.synchronize()
        st = chem.integrate_boxes(boxes, rtol=1e-9, atol=1e-20)
    print(label, "bulk_ms %.2f sparse_ms %.2f att %d iters %d" % (st["t_bulk_ms"], st["t_sparse_ms"], st["steps_attempted"], st["bulk_iters"]))

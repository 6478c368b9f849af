import sys, os, time, json
sys.path.insert(0, os.getcwd())
import torch, numpy as np, synth, bench
from paper_2510_23993_b200 import Box, Chem
dev = torch.device("cuda", 0)
doc = synth.load_trajectories()
chem = Chem("h2air_li2004", device=0, atol_T=1e-6)
raw, _ = synth.field_cfg2(doc, side=64, box=64, device=dev)   # 262144 identical cells, 1 box
b = raw[0]
box = Box(b["rho"], chem.energy(b["T"], b["Y"]), b["T"].clone(), b["Y"].clone(), 1e-7)
T0, Y0 = box.T.clone(), box.Y.clone()
for ns, label in ((10**4, "bulk"), (10**9, "sparse-only")):
    chem.set_opts(n_active_star=ns)
    for rep in range(3):
        box.T.copy_(T0); box.Y.copy_(Y0); torch.cuda.synchronize()
        st = chem.integrate_boxes([box], rtol=1e-9, atol=1e-20)
    print(label, "bulk_ms", st["t_bulk_ms"], "sparse_ms", st["t_sparse_ms"], "att", st["steps_attempted"], "rhs", st["rhs_evals"])

#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over a small chem_integrate
# (cfg1c cells in two boxes: the free-running, lockstep, cross-call and in-call heavy-first launches, budget-capped calls).  Output: gpurun_out/sanitize_*.txt
mkdir -p gpurun_out
cat > /tmp/san_case.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth
from paper_2510_23993_b200 import Chem, Box
from paper_2510_23993_b200 import load_mechanism
m = load_mechanism("h2air_li2004")
d = synth.cfg1c(m.species, m.W)
idx = np.arange(0, 4096, 64)
dev = torch.device("cuda", 0)
for lock, lpt, ksp in ((0, 0, 100000), (1, 0, 100000), (0, 1, 100000), (0, 1, 7), (0, 0, 7), (0, 3, 100000), (0, 3, 7), (2, 2, 100000)):
    ch = Chem("h2air_li2004", device=0, kmax_bulk=3, n_active_star=16, lockstep=lock, schedule_lpt=lpt,
              kmax_sparse=ksp)
    T = torch.tensor(d["T"][idx], device=dev)
    Y = torch.tensor(d["Y"][idx].T.copy(), device=dev)
    rho = torch.tensor(d["rho"][idx], device=dev)
    e = ch.energy(T, Y)
    cost = torch.zeros(2, dtype=torch.float64, device=dev)
    n = len(idx) // 2
    boxes = [Box(rho[:n], e[:n], T[:n].clone(), Y[:, :n].contiguous(), 1e-6),
             Box(rho[n:], e[n:], T[n:].clone(), Y[:, n:].contiguous(), 1e-5)]
    st = ch.integrate_boxes(boxes, box_cost=cost)
    w = ch.rates(rho, T, Y)
    J = ch.jacobian(rho[:8], T[:8], Y[:, :8].contiguous())
    torch.cuda.synchronize()
    st2 = ch.integrate_boxes(boxes, box_cost=cost)      # second call: cost hints from the first
    torch.cuda.synchronize()
    status, steps = ch.cell_status(substeps=True)
    torch.cuda.synchronize()
    print("lockstep", lock, "lpt", lpt, "kmax_sparse", ksp, st["steps_attempted"], st["sparse_cells"], st2["lpt"],
          int(status.sum()), int(steps.sum()))
PY
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python /tmp/san_case.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$tool.txt | tail -1)"
done

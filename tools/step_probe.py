"""Step-size sequence probe (GPU): for sampled cells of a config, the local time t and the next substep
h after k = 1..K attempted substeps (sparse-only calls with kmax_sparse = k, read from the workspace),
so one can see whether the first substep or the x6 growth cap limits the step count.

    python tools/step_probe.py cfg2 [K]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2510_23993_b200 import Chem  # noqa: E402


def cells(cfg, n):
    doc = synth.load_trajectories()
    if cfg == "cfg2":
        tr = next(t for t in doc["trajectories"] if t["kind"] == "fresh" and t["T0"] == 1200.0)
        r, T, Y = synth.traj_state(tr, 0.9)
        return np.full(n, r), np.full(n, T), np.tile(Y, (n, 1)), 1e-7
    d = synth.cfg1b(doc, n=n)
    return d["rho"], d["T"], d["Y"], d["dt"]


def main(cfg="cfg2", K=6, n=4096, h0=0.01):
    chem = Chem("h2air_li2004", device=0, n_active_star=10 ** 12, h0_factor=h0)
    rho, T0, Y, dt = cells(cfg, n)
    dev = torch.device("cuda", 0)
    rho_d = torch.tensor(rho, device=dev)
    e_d = chem.energy(torch.tensor(T0, device=dev), torch.tensor(Y.T.copy(), device=dev))
    al = lambda x: (x + 255) & ~255
    for k in range(1, K + 1):
        Td = torch.tensor(T0, device=dev)
        Yd = torch.tensor(Y.T.copy(), device=dev)
        chem.set_opts(kmax_sparse=k)
        st = chem.integrate(rho_d, e_d, Td, Yd, dt, rtol=1e-9, atol=1e-20)
        torch.cuda.synchronize()
        ws = chem._ws
        o = al(al(al(15 * 8) + 56) + 16)
        t = ws[o:o + 8 * n].view(torch.float64).cpu().numpy()
        o2 = al(o + 8 * n)
        h = ws[o2:o2 + 8 * n].view(torch.float64).cpu().numpy()
        print(f"{cfg} h0={h0} k={k}: t/dt median {np.median(t) / dt:.4g} min {t.min() / dt:.4g}  next h/dt median "
              f"{np.median(h) / dt:.4g}  attempted {st['steps_attempted']} accepted {st['steps_accepted']} "
              f"unfinished {st['n_unfinished']}", flush=True)


if __name__ == "__main__":
    for c in (sys.argv[1:] or ["cfg2", "cfg1b"]):
        for h0 in (0.01, 0.03):
            main(c, 6, h0=h0)

"""Bitwise comparison of two libchem builds on the same inputs: integrate cfg1b cells (radical-rich,
stiff) and a slice of the cfg3 detonation field with the build in place and write T, Y to an .npz;
run once per build, then compare.

    python tools/bitwise_builds.py out_a.npz ; (swap libchem.so) ; python tools/bitwise_builds.py out_b.npz
    python tools/bitwise_builds.py --compare out_a.npz out_b.npz
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(out):
    import torch

    import synth
    from oracle import Oracle
    from paper_2510_23993_b200 import Chem
    ora = Oracle("h2air_li2004")
    m = ora.m
    chem = Chem("h2air_li2004", device=0)
    res = {}
    for name, d in (("cfg1b", synth.cfg1b(synth.load_trajectories(), n=4096)),
                    ("cfg1c", synth.cfg1c(m.species, m.W))):
        e = np.array([ora.energy(t, y) for t, y in zip(d["T"], d["Y"])])
        T = torch.tensor(d["T"], dtype=torch.float64, device="cuda")
        Y = torch.tensor(d["Y"].T.copy(), dtype=torch.float64, device="cuda")
        rho = torch.tensor(d["rho"], dtype=torch.float64, device="cuda")
        st = chem.integrate(rho, torch.tensor(e, device="cuda"), T, Y, d["dt"], rtol=1e-9, atol=1e-20)
        res[name + "_T"] = T.cpu().numpy()
        res[name + "_Y"] = Y.cpu().numpy()
        res[name + "_steps"] = np.array([st["steps_attempted"]])
    np.savez(out, **res)


def compare(a, b):
    A, B = np.load(a), np.load(b)
    ok = True
    for k in A.files:
        same = np.array_equal(A[k], B[k])
        ok &= same
        print(k, "bitwise equal" if same else f"DIFFER (max abs {np.max(np.abs(A[k] - B[k])):.3e})")
    print("ALL BITWISE EQUAL" if ok else "BUILDS DIFFER")


if __name__ == "__main__":
    if sys.argv[1] == "--compare":
        compare(sys.argv[2], sys.argv[3])
    else:
        run(sys.argv[1])

"""Micro-benchmarks of the point kernels (rates, rhs, jacobian, energy) and an FP64 DFMA peak probe.

    python tools/micro.py            (on a GPU box)

Prints one JSON line per kernel: cells/s and achieved algorithmic FP64 TFLOP/s (flops.py model).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2510_23993_b200 import Chem  # noqa: E402
from paper_2510_23993_b200.flops import FlopModel  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) / 1e3)
    return min(ts)


def main():
    dev = torch.device("cuda", 0)
    chem = Chem("h2air_li2004", device=0)
    fm = FlopModel(chem.mech)
    n = int(os.environ.get("MICRO_N", 1 << 22))
    d = synth.cfg1d(chem.mech.species, chem.mech.W, n=4096)
    idx = np.arange(n) % 4096
    rho = torch.tensor(d["rho"][idx], device=dev)
    T = torch.tensor(d["T"][idx], device=dev)
    Y = torch.tensor(d["Y"][idx].T.copy(), device=dev)
    out = torch.empty((chem.ns + 1, n), dtype=torch.float64, device=dev)
    res = {}
    t = timeit(lambda: chem.rates(rho, T, Y, out=out[: chem.ns]))
    res["rates"] = dict(s=t, cells_per_s=n / t, tflops=n * fm.rhs / t / 1e12)
    t = timeit(lambda: chem.rhs(rho, T, Y, out=out))
    res["rhs"] = dict(s=t, cells_per_s=n / t, tflops=n * fm.rhs / t / 1e12)
    m = n // 8
    t = timeit(lambda: chem.jacobian(rho[:m], T[:m], Y[:, :m]))
    res["jacobian(full, FULL=true)"] = dict(s=t, cells_per_s=m / t, tflops=m * (fm.jac + fm.rhs) / t / 1e12)
    t = timeit(lambda: chem.energy(T, Y, out=out[0]))
    res["energy"] = dict(s=t, cells_per_s=n / t, GBps=n * (8 * 10 + 8) / t / 1e9)
    for k, v in res.items():
        print(json.dumps({"kernel": k, **v}))


if __name__ == "__main__":
    main()

"""Per-call host overhead of chem_integrate_boxes (GPU): wall time of N calls on a tiny field
(one box of 32 cfg1 cells), the floor every fused call pays (gate, counter reads, launches, stats)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2510_23993_b200 import Box, Chem, load_mechanism  # noqa: E402

m = load_mechanism("h2air_li2004")
d = synth.cfg1(m.species, m.W)
dev = torch.device("cuda", 0)
chem = Chem("h2air_li2004", device=0)
idx = np.arange(32)
T0 = torch.tensor(d["T"][idx], device=dev)
Y0 = torch.tensor(d["Y"][idx].T.copy(), device=dev)
rho = torch.tensor(d["rho"][idx], device=dev)
e = chem.energy(T0, Y0)
for nb in (1, 16):
    boxes = [Box(rho, e, T0.clone(), Y0.clone(), 1e-9) for _ in range(nb)]
    for _ in range(5):
        chem.integrate_boxes(boxes)
    torch.cuda.synchronize()
    t = time.perf_counter()
    N = 200
    for _ in range(N):
        chem.integrate_boxes(boxes)
    torch.cuda.synchronize()
    print(f"boxes={nb}: {1e6 * (time.perf_counter() - t) / N:.1f} us per integrate_boxes call (wall)")

# split: Python marshalling vs the C call
import ctypes  # noqa: E402
from paper_2510_23993_b200 import binding as _b  # noqa: E402
boxes = [Box(rho, e, T0.clone(), Y0.clone(), 1e-9) for _ in range(16)]
chem.integrate_boxes(boxes)
arr = (_b.ChemBox * 16)()
for i, bx in enumerate(boxes):
    arr[i].rho, arr[i].e, arr[i].T, arr[i].Y = bx.rho.data_ptr(), bx.e.data_ptr(), bx.T.data_ptr(), bx.Y.data_ptr()
    arr[i].solid, arr[i].ncells, arr[i].ld, arr[i].dt = None, bx.ncells, bx.Y.stride(0), 1e-9
ws = chem.workspace(32 * 16, 16)
st = _b.ChemStats()
strm = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(200):
    chem.lib.chem_integrate_boxes(chem._h, 16, arr, 1e-9, 1e-20, ctypes.c_void_p(ws.data_ptr()), ws.numel(), None,
                                  ctypes.byref(st), strm)
torch.cuda.synchronize()
print(f"raw C call: {1e6 * (time.perf_counter() - t) / 200:.1f} us")
t = time.perf_counter()
for _ in range(2000):
    torch.cuda.synchronize()
print(f"torch.cuda.synchronize round trip: {1e6 * (time.perf_counter() - t) / 2000:.1f} us")

"""Seeded synthetic input generators shared by the tests, the bench and the oracle baseline.

This module holds NONE of the method's arithmetic (no thermo, no rates, no integration): it
produces (rho, T, Y) fields with the shapes, value distributions and structure of the paper's
workloads (SURVEY.md §8(d) recipes; BASELINE.json configs), plus table look-ups into
data/trajectories_*.json, which a committed script (tools/make_trajectories.py) wrote by calling
only oracle/.  The internal energy e = u(T0, Y) that the method takes as input is evaluated by
each side with its own thermo (the CUDA path: chem_energy; the oracle: or_energy).

Conventions: species order H2, O2, H2O, H, O, OH, HO2, H2O2, N2; phi = 1 H2-air
with O2:N2 = 1:3.76 by moles; rho = p Wbar/(R T) (ideal-gas input recipe); dt = 1e-7 s; seed =
23993 + config index.
"""
from __future__ import annotations

import json
import pathlib

import numpy as np

R_GAS = 8.314462618
P_ATM = 101325.0
DATA = pathlib.Path(__file__).resolve().parent.parent / "data"
SEED0 = 23993


def fresh_Y(species, W, phi=1.0):
    """Mass fractions of phi-equivalence H2-air (SURVEY reading 18)."""
    X = np.zeros(len(species))
    X[species.index("H2")] = 2.0 * phi
    X[species.index("O2")] = 1.0
    X[species.index("N2")] = 3.76
    Y = X * np.asarray(W)
    return Y / Y.sum()


def air_Y(species, W):
    X = np.zeros(len(species))
    X[species.index("O2")] = 1.0
    X[species.index("N2")] = 3.76
    Y = X * np.asarray(W)
    return Y / Y.sum()


def rho_ideal(p, T, Y, W):
    """Input recipe: rho = p Wbar / (R T), Wbar = 1/sum(Y/W)."""
    Y = np.atleast_2d(Y)
    return np.asarray(p) / (R_GAS * np.asarray(T) * np.sum(Y / np.asarray(W)[None, :], axis=1))


def cfg1(species, W, dt=1e-7, n=4096):
    """configs[0]: n independent 0-D reactors, T0_i = 900 + 600 i/(n-1) K, 1 atm, fresh phi=1."""
    T = 900.0 + 600.0 * np.arange(n) / max(n - 1, 1)
    Y = np.tile(fresh_Y(species, W), (n, 1))
    rho = rho_ideal(P_ATM, T, Y, W)
    return dict(rho=rho, T=T, Y=Y, dt=dt, name="cfg1")


def cfg1c(species, W):
    """Companion parity set 1c: the cfg1 cells with dt = 1e-4 s (ignition inside the step)."""
    d = cfg1(species, W, dt=1e-4)
    d["name"] = "cfg1c"
    return d


def cfg1d(species, W, n=4096, seed=SEED0 + 100):
    """Companion set 1d (rates only): T ~ U[300,3000] K, p ~ logU[0.1,100] atm, Y ~ Dirichlet(0.5)
    with 20% of entries zeroed, then renormalised."""
    rng = np.random.Generator(np.random.PCG64(seed))
    ns = len(species)
    T = rng.uniform(300.0, 3000.0, n)
    p = P_ATM * 10.0 ** rng.uniform(-1.0, 2.0, n)
    Y = rng.dirichlet(0.5 * np.ones(ns), n)
    Y[rng.random((n, ns)) < 0.2] = 0.0
    empty = Y.sum(1) == 0
    Y[empty, -1] = 1.0
    Y /= Y.sum(1, keepdims=True)
    rho = rho_ideal(p, T, Y, W)
    return dict(rho=rho, T=T, Y=Y, dt=None, name="cfg1d")


# ------------------------------------------------------------------ trajectory tables
def load_trajectories(name="trajectories_h2air_li2004"):
    """Oracle-written table of 0-D constant-volume trajectories (see tools/make_trajectories.py)."""
    path = DATA / f"{name}.json"
    doc = json.loads(path.read_text())
    for tr in doc["trajectories"]:
        tr["t_over_tau"] = np.array(tr["t_over_tau"])
        tr["T"] = np.array(tr["T"])
        tr["Y"] = np.array(tr["Y"])
    return doc


def traj_state(tr, frac):
    """Nearest stored state at t/tau = frac (table look-up, no interpolation)."""
    i = np.clip(np.searchsorted(tr["t_over_tau"], frac), 0, len(tr["t_over_tau"]) - 1)
    j = np.maximum(i - 1, 0)
    pick = np.where(np.abs(tr["t_over_tau"][j] - frac) <= np.abs(tr["t_over_tau"][i] - frac), j, i)
    return tr["rho"], tr["T"][pick], tr["Y"][pick]


def cfg1b(doc, n=4096, seed=SEED0 + 101, dt=1e-7):
    """Companion set 1b: reactor-trajectory states from T0 in {1000..1500} K at t/tau ~ U[0.5, 1.5]
    (radical-rich, stiff), dt = 1e-7."""
    rng = np.random.Generator(np.random.PCG64(seed))
    trs = [t for t in doc["trajectories"] if t["kind"] == "fresh" and 1000.0 <= t["T0"] <= 1500.0]
    which = rng.integers(0, len(trs), n)
    frac = rng.uniform(0.5, 1.5, n)
    rho = np.empty(n); T = np.empty(n); Y = np.empty((n, len(doc["species"])))
    for i in range(n):
        r, t, y = traj_state(trs[which[i]], frac[i])
        rho[i], T[i], Y[i] = r, t, y
    return dict(rho=rho, T=T, Y=Y, dt=dt, name="cfg1b")


# ------------------------------------------------------------------ device fields (torch)
def _state_boxes(rho, T, Y, nboxes, ncell, device):
    """nboxes boxes of ncell identical cells (component-major Y [ns, ncell] per box)."""
    import torch
    out = []
    for _ in range(nboxes):
        out.append(dict(
            rho=torch.full((ncell,), float(rho), dtype=torch.float64, device=device),
            T=torch.full((ncell,), float(T), dtype=torch.float64, device=device),
            Y=torch.as_tensor(np.asarray(Y, dtype=np.float64), device=device)[:, None].expand(-1, ncell).contiguous()))
    return out


def field_cfg2(doc, side=128, box=32, device="cuda", dt=1e-7):
    """configs[1]: uniform side^3 field, every cell the same reactor-trajectory state (T0 = 1200 K,
    1 atm, phi = 1, at t = 0.9 tau_ign: mid-induction, stiff), as (side/box)^3 boxes of box^3."""
    tr = next(t for t in doc["trajectories"] if t["kind"] == "fresh" and t["T0"] == 1200.0)
    rho, T, Y = traj_state(tr, 0.9)
    nb = (side // box) ** 3
    boxes = _state_boxes(rho, T, Y, nb, box ** 3, device)
    for b in boxes:
        b["dt"] = dt
    meta = dict(workload=f"cfg2: uniform {side}^3 H2-air field, T0=1200 K traj. state at t=0.9 tau, "
                         f"{nb} boxes of {box}^3, dt={dt:g} s", cells=side ** 3, state=dict(rho=float(rho),
                T=float(T), Y=np.asarray(Y).tolist()))
    return boxes, meta


def field_cfg2b(doc, side=128, box=32, device="cuda", dt=1e-7, seed=SEED0 + 12):
    """configs[1] variant 2b: the cfg2 field with every cell's trajectory time drawn
    per cell, t/tau ~ U[0.85, 0.95] (counter-based hash of the global cell index), so neighbouring
    cells need different substep counts (intra-warp divergence on an otherwise uniform field)."""
    import torch
    tab = _traj_tables(doc, "fresh", device, T0=1200.0)
    nb1 = side // box
    n = box ** 3
    boxes = []
    for b in range(nb1 ** 3):
        gidx = torch.arange(b * n, (b + 1) * n, device=device, dtype=torch.int64)
        frac = 0.85 + 0.1 * hash_uniform(gidx, seed)
        T, Y = _lookup(tab, frac)
        boxes.append(dict(rho=torch.full((n,), tab["rho"], dtype=torch.float64, device=device), T=T.clone(),
                          Y=Y.T.contiguous(), dt=dt))
    meta = dict(workload=f"cfg2b: {side}^3 H2-air field, T0=1200 K traj. states at t/tau ~ U[0.85, 0.95] per cell, "
                         f"{nb1 ** 3} boxes of {box}^3, dt={dt:g} s", cells=side ** 3)
    return boxes, meta


# ------------------------------------------------------------------ counter-based randomness
def hash_uniform(idx, seed):
    """Uniform [0, 1) from a 32-bit integer hash of (idx, seed); idx is an int64 torch tensor.
    A pure function of its arguments, so any rank/box can regenerate any cell."""
    import torch
    M32 = 0xFFFFFFFF
    x = (idx.to(torch.int64) * 0x9E3779B1 + (seed & M32) * 0x7F4A7C15 + 0x165667B1) & M32
    for mul in (0x7FEB352D, 0x2C1B3C6D, 0x297A2D39):       # multipliers < 2^31: products fit int64
        x = x ^ (x >> 16)
        x = (x * mul) & M32
    x = x ^ (x >> 15)
    return x.to(torch.float64) / 4294967296.0


def _traj_tables(doc, kind, device, **sel):
    """Stack a trajectory's samples into device tensors (T [m], Y [m, ns], rho scalar, dfrac)."""
    import torch
    tr = next(t for t in doc["trajectories"] if t["kind"] == kind and all(t.get(k) == v for k, v in sel.items()))
    fr = tr["t_over_tau"]
    return dict(T=torch.as_tensor(tr["T"], dtype=torch.float64, device=device),
                Y=torch.as_tensor(tr["Y"], dtype=torch.float64, device=device),
                rho=float(tr["rho"]), frac0=float(fr[0]), dfrac=float(fr[1] - fr[0]), m=len(fr), tau=tr["tau"])


def _lookup(tab, frac):
    """Nearest stored sample of a uniformly sampled trajectory (no interpolation)."""
    import torch
    i = torch.clamp(torch.round((frac - tab["frac0"]) / tab["dfrac"]), 0, tab["m"] - 1).to(torch.int64)
    return tab["T"][i], tab["Y"][i]


def detonation_box(doc, W, species, lo, shape, level, seed, device, x_front=5.0, amp=2.0, period=64.0,
                   phase=0.0, spots=None):
    """One box of a detonation-shaped field (cfg3 / cfg4 recipe).

    Coordinates in level-0 cell units: cell (i, j, k) of a level-l box at position
    ((lo + idx) + 0.5) / 2^l.  Cold fresh gas (300 K, 1 atm, phi = 1) except (i) a detonation band
    x < x_f(y) = x_front + amp sin(2 pi y/period + phase) holding the von Neumann trajectory
    state at t/tau_vN = 3 d/x_f (d = x_f - x), and (ii) perturbation spheres of radius 3 at
    1500 K, 1 atm.  Layout: x fastest (AMReX Fortran order).  Returns dict(rho, T, Y[ns, n])."""
    import torch
    nx, ny, nz = shape
    s = 0.5 ** level
    i = torch.arange(nx, device=device, dtype=torch.float64)
    j = torch.arange(ny, device=device, dtype=torch.float64)
    k = torch.arange(nz, device=device, dtype=torch.float64)
    z3, y3, x3 = torch.meshgrid(k, j, i, indexing="ij")            # x fastest after flatten
    x = ((lo[0] + x3) + 0.5) * s
    y = ((lo[1] + y3) + 0.5) * s
    z = ((lo[2] + z3) + 0.5) * s
    x, y, z = x.reshape(-1), y.reshape(-1), z.reshape(-1)
    n = x.numel()
    ns = len(species)
    Yf = torch.as_tensor(fresh_Y(species, W), dtype=torch.float64, device=device)
    Wt = torch.as_tensor(np.asarray(W), dtype=torch.float64, device=device)
    T = torch.full((n,), 300.0, dtype=torch.float64, device=device)
    Y = Yf[None, :].expand(n, ns).clone()
    rho_f = lambda Tv: P_ATM / (R_GAS * Tv * torch.sum(Yf / Wt))      # noqa: E731 (ideal-gas recipe)
    rho = rho_f(T)
    xf = x_front + amp * torch.sin(2 * np.pi * y / period + phase)
    band = x < xf
    if band.any():
        vn = _traj_tables(doc, "vN", device)
        Tb, Yb = _lookup(vn, 3.0 * (xf[band] - x[band]) / xf[band])
        T[band] = Tb
        Y[band] = Yb
        rho[band] = vn["rho"]
    for (cx, cy, cz) in (spots or []):
        sp = (x - cx) ** 2 + (y - cy) ** 2 + (z - cz) ** 2 < 9.0
        sp &= ~band
        if sp.any():
            T[sp] = 1500.0
            Y[sp] = Yf
            rho[sp] = rho_f(torch.full_like(T[sp], 1500.0))
    return dict(rho=rho, T=T, Y=Y.t().contiguous())


def spot_centres(seed, n=8, side=256.0):
    """cfg3: 8 perturbation spheres at seeded x in [16, 48] (P:336 'perturbation zones slightly
    downstream' of the driver), y, z uniform over the domain."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return [(float(rng.uniform(16, 48)), float(rng.uniform(0, side)), float(rng.uniform(0, side))) for _ in range(n)]


def field_cfg3(doc, W, species, side=256, box=64, device="cuda", dt=1e-7, seed=SEED0 + 2, box_ids=None):
    """configs[2]: side^3 detonation-shaped field (~2% active), boxes of box^3.  box_ids selects a
    subset of the (side/box)^3 boxes (multi-GPU sharding / sampled parity)."""
    nb1 = side // box
    spots = spot_centres(seed, side=float(side))
    ids = range(nb1 ** 3) if box_ids is None else box_ids
    out = []
    for b in ids:
        bi, bj, bk = b % nb1, (b // nb1) % nb1, b // (nb1 * nb1)
        d = detonation_box(doc, W, species, (bi * box, bj * box, bk * box), (box, box, box), 0, seed, device,
                           spots=spots)
        d.update(dt=dt, box_id=b)
        out.append(d)
    meta = dict(workload=f"cfg3: {side}^3 detonation-shaped H2-air field (band x<5+2sin(2pi y/64) at vN "
                         f"trajectory states + 8 hot spots, cold 300 K elsewhere), {nb1 ** 3} boxes of {box}^3, "
                         f"dt={dt:g} s", cells=side ** 3)
    return out, meta


def hierarchy_cfg4(copy, nboxes_level=64, box=32, dt=1e-7, seed=SEED0 + 3):
    """configs[3] box list of one copy (rank p owns copy p before balancing): 3 levels, ratio 2,
    32^3 boxes.  L0: 128^3 (64 boxes); L1: 64 boxes covering the 1/8 of L0 at the front
    ([0,64)^3 L0 cells); L2: 64 boxes covering [0,32)^3 L0 cells.  Subcycling: level l
    integrates over dt/2^l, 2^l times per coarse step.  Returns [(copy, level, box_index, lo, dt)]."""
    out = []
    for level in range(3):
        for b in range(nboxes_level):
            bi, bj, bk = b % 4, (b // 4) % 4, b // 16
            out.append(dict(copy=copy, level=level, index=b, lo=(bi * box, bj * box, bk * box),
                            shape=(box, box, box), dt=dt / 2 ** level))
    return out


def cfg4_copy_params(copy, seed=SEED0 + 3):
    """Per-copy seed: front phase and spot positions differ between copies (so per-copy costs differ)."""
    rng = np.random.Generator(np.random.PCG64(seed + 1000 * copy))
    phase = float(rng.uniform(0, 2 * np.pi))
    spots = [(float(rng.uniform(16, 48)), float(rng.uniform(0, 128)), float(rng.uniform(0, 128))) for _ in range(8)]
    return phase, spots


def build_cfg4_box(doc, W, species, desc, device):
    phase, spots = cfg4_copy_params(desc["copy"])
    d = detonation_box(doc, W, species, desc["lo"], desc["shape"], desc["level"], 0, device, phase=phase,
                       spots=spots)
    d.update(dt=desc["dt"])
    return d


def jisc_box(doc, W, species, lo, shape, seed, device, jet=(64.0, 128.0), d_jet=8.0, Z_st=0.0285):
    """One box of the jet-in-crossflow-shaped field (configs[4], SURVEY.md §8(d) cfg5 recipe):
    x streamwise, y span, z wall-normal; air crossflow at 1200 K; H2 jet at 250 K from (x_j, y_j);
    plume centreline z_c = 2d((x-x_j)/d)^(1/3), half-width sigma = 0.5d + 0.1(x-x_j) with +-10%
    seeded noise; Z = exp(-r^2/2 sigma^2) min(1, 3d/(x-x_j+3d)); the mixed state (Y, h linear in Z
    at 1 atm) from the oracle-written mixing table; shear-layer cells (|Z - Z_st| < 0.01,
    T_mix >= 900 K) take reactor-trajectory states of the mixed gas at t ~ U[0, 2] tau."""
    import torch
    mix = doc["jisc_mixing"]
    Zt = torch.as_tensor(mix["Z"], dtype=torch.float64, device=device)
    Tt = torch.as_tensor(mix["T"], dtype=torch.float64, device=device)
    Rt = torch.as_tensor(mix["rho"], dtype=torch.float64, device=device)
    Yj = torch.as_tensor(mix["Y_jet"], dtype=torch.float64, device=device)
    Ya = torch.as_tensor(mix["Y_air"], dtype=torch.float64, device=device)
    nx, ny, nz = shape
    i = torch.arange(nx, device=device, dtype=torch.float64)
    j = torch.arange(ny, device=device, dtype=torch.float64)
    k = torch.arange(nz, device=device, dtype=torch.float64)
    z3, y3, x3 = torch.meshgrid(k, j, i, indexing="ij")
    x = (lo[0] + x3 + 0.5).reshape(-1)
    y = (lo[1] + y3 + 0.5).reshape(-1)
    z = (lo[2] + z3 + 0.5).reshape(-1)
    xj, yj = jet
    dx = x - xj
    down = dx > 0
    xcol = torch.floor(x).to(torch.int64)
    noise = 1.0 + 0.1 * (2.0 * hash_uniform(xcol, seed) - 1.0)
    sigma = (0.5 * d_jet + 0.1 * torch.clamp(dx, min=0.0)) * noise
    zc = 2.0 * d_jet * torch.pow(torch.clamp(dx, min=0.0) / d_jet, 1.0 / 3.0)
    r2 = (y - yj) ** 2 + (z - zc) ** 2
    Z = torch.exp(-r2 / (2 * sigma ** 2)) * torch.clamp(3 * d_jet / (torch.clamp(dx, min=0.0) + 3 * d_jet), max=1.0)
    # the jet column itself (x near x_j, below the plume): pure jet fluid within d/2 of the axis
    col = (dx.abs() <= d_jet / 2) & ((y - yj) ** 2 + dx ** 2 <= (d_jet / 2) ** 2) & (z <= zc + d_jet)
    Z = torch.where(down | col, Z, torch.zeros_like(Z))
    Z = torch.where(col, torch.ones_like(Z), Z)
    iz = torch.clamp(torch.round(Z * (len(mix["Z"]) - 1)), 0, len(mix["Z"]) - 1).to(torch.int64)
    T = Tt[iz].clone()
    rho = Rt[iz].clone()
    Zq = Zt[iz]
    Y = (Zq[:, None] * Yj[None, :] + (1 - Zq[:, None]) * Ya[None, :])
    shear = ((Zq - Z_st).abs() < 0.01) & (T >= 900.0)
    if shear.any():
        trs = [t for t in doc["trajectories"] if t["kind"] == "jisc_shear"]
        zs = torch.as_tensor([t["Z"] for t in trs], dtype=torch.float64, device=device)
        which = torch.argmin((Zq[shear][:, None] - zs[None, :]).abs(), dim=1)
        gidx = ((z * 4096 + y) * 4096 + x).to(torch.int64)[shear]
        frac = 2.0 * hash_uniform(gidx, seed + 7)
        Ts = torch.empty_like(frac)
        Ys = torch.empty((frac.numel(), Y.shape[1]), dtype=torch.float64, device=device)
        Rs = torch.empty_like(frac)
        for w, tr in enumerate(trs):
            sel = which == w
            if sel.any():
                tab = _traj_tables(doc, "jisc_shear", device, Z=tr["Z"])
                a, bY = _lookup(tab, frac[sel])
                Ts[sel] = a
                Ys[sel] = bY
                Rs[sel] = tab["rho"]
        T[shear] = Ts
        Y[shear] = Ys
        rho[shear] = Rs
    return dict(rho=rho, T=T, Y=Y.t().contiguous())


def field_cfg5(doc, W, species, shape=(512, 256, 256), box=64, device="cuda", dt=1e-7, seed=SEED0 + 4,
               box_ids=None):
    """configs[4]: 512x256x256 jet-in-crossflow-shaped field, 128 boxes of 64^3 (8 x 4 x 4)."""
    nbx, nby, nbz = shape[0] // box, shape[1] // box, shape[2] // box
    ids = range(nbx * nby * nbz) if box_ids is None else box_ids
    out = []
    for b in ids:
        bi, bj, bk = b % nbx, (b // nbx) % nby, b // (nbx * nby)
        d = jisc_box(doc, W, species, (bi * box, bj * box, bk * box), (box, box, box), seed, device)
        d.update(dt=dt, box_id=b)
        out.append(d)
    meta = dict(workload=f"cfg5: {shape[0]}x{shape[1]}x{shape[2]} jet-in-crossflow-shaped H2-air field, "
                         f"{nbx * nby * nbz} boxes of {box}^3, dt={dt:g} s", cells=int(np.prod(shape)))
    return out, meta

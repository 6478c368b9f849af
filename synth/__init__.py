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

"""Oracle-side mechanism loader (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Reads a mechanism YAML file from mech/ into plain numpy arrays in SI-molar units and checks
the invariants SPEC.md states for a mechanism (S:24 contiguous thermo ranges, S:28 mass and
element balance per reaction, W > 0).  This loader shares no code with the product's loader
(paper_2510_23993_b200/mechanism.py); only the data file is shared.
"""
from __future__ import annotations

import dataclasses
import pathlib

import numpy as np
import yaml

R_GAS = 8.314462618          # J/(mol K)   (SURVEY.md §8(a) A4 block)
P_REF = 101325.0             # Pa          (CHEMKIN standard-state convention, SURVEY reading 6)
CAL = 4.184                  # J/cal

KIND_ELEMENTARY, KIND_THREEBODY, KIND_LINDEMANN, KIND_TROE = 0, 1, 2, 3

MECH_DIR = pathlib.Path(__file__).resolve().parent.parent / "mech"


@dataclasses.dataclass
class OracleMechanism:
    name: str
    species: list
    elements: list
    W: np.ndarray            # [ns] kg/mol
    comp: np.ndarray         # [ns, ne] atom counts
    T_range: np.ndarray      # [ns, 3]
    nasa_lo: np.ndarray      # [ns, 7]
    nasa_hi: np.ndarray      # [ns, 7]
    nu_f: np.ndarray         # [nr, ns] int  reactant coefficients nu'
    nu_r: np.ndarray         # [nr, ns] int  product coefficients nu''
    A: np.ndarray            # [nr] SI (k_inf for falloff rows)
    b: np.ndarray
    Ea: np.ndarray           # J/mol
    kind: np.ndarray         # [nr] int
    reversible: np.ndarray   # [nr] int
    eff: np.ndarray          # [nr, ns] third-body efficiencies (1 default)
    A0: np.ndarray           # [nr] low-pressure limit (falloff rows)
    b0: np.ndarray
    Ea0: np.ndarray
    troe: np.ndarray         # [nr, 4] alpha, T***, T*, T** (T** <= 0: term absent)

    @property
    def ns(self):
        return len(self.species)

    @property
    def nr(self):
        return self.A.shape[0]


def _length_factor(units):
    return {"cm": 1e-2, "m": 1.0}[units.get("length", "m")]


def _energy_factor(units):
    return {"cal/mol": CAL, "J/mol": 1.0, "kcal/mol": 1000 * CAL}[units.get("activation-energy", "J/mol")]


def load(name_or_path) -> OracleMechanism:
    p = pathlib.Path(name_or_path)
    if not p.exists():
        p = MECH_DIR / f"{name_or_path}.yaml"
    doc = yaml.safe_load(p.read_text())
    units = doc.get("units", {})
    L = _length_factor(units)
    conc = L ** 3            # (cm^3/mol) -> (m^3/mol)
    eF = _energy_factor(units)
    aw = doc["atomic_weights"]
    elements = list(aw.keys())
    sp = doc["species"]
    names = [s["name"] for s in sp]
    if len(set(names)) != len(names):
        raise ValueError("duplicate species names")
    ns, ne = len(sp), len(elements)
    comp = np.zeros((ns, ne), dtype=np.int64)
    for k, s in enumerate(sp):
        for el, cnt in s["composition"].items():
            comp[k, elements.index(el)] = cnt
    W = comp @ np.array([aw[e] for e in elements], dtype=np.float64) * 1e-3
    if np.any(W <= 0):
        raise ValueError("W must be > 0")
    T_range = np.array([s["T_range"] for s in sp], dtype=np.float64)
    if np.any(T_range[:, 0] >= T_range[:, 1]) or np.any(T_range[:, 1] >= T_range[:, 2]):
        raise ValueError("thermo ranges must be ordered and contiguous")
    lo = np.array([s["low"] for s in sp], dtype=np.float64)
    hi = np.array([s["high"] for s in sp], dtype=np.float64)

    rx = doc["reactions"]
    nr = len(rx)
    nu_f = np.zeros((nr, ns), dtype=np.int64)
    nu_r = np.zeros((nr, ns), dtype=np.int64)
    A = np.zeros(nr); b = np.zeros(nr); Ea = np.zeros(nr)
    A0 = np.zeros(nr); b0 = np.zeros(nr); Ea0 = np.zeros(nr)
    kind = np.zeros(nr, dtype=np.int64)
    rev = np.ones(nr, dtype=np.int64)
    eff = np.ones((nr, ns))
    troe = np.zeros((nr, 4))
    for r, x in enumerate(rx):
        for s, v in x["reactants"].items():
            nu_f[r, names.index(s)] += int(v)
        for s, v in x["products"].items():
            nu_r[r, names.index(s)] += int(v)
        order = int(nu_f[r].sum())
        t = x.get("type", "elementary")
        rev[r] = 1 if x.get("reversible", True) else 0
        if t == "elementary":
            kind[r] = KIND_ELEMENTARY
            rate = x["rate"]
            A[r] = rate["A"] * conc ** (order - 1)
        elif t == "three-body":
            kind[r] = KIND_THREEBODY
            rate = x["rate"]
            A[r] = rate["A"] * conc ** order           # M adds one to the order
        elif t == "falloff":
            rate = x["high"]
            lowr = x["low"]
            A[r] = rate["A"] * conc ** (order - 1)       # k_inf
            A0[r] = lowr["A"] * conc ** order            # k_0 multiplies [M]
            b0[r] = lowr["b"]
            Ea0[r] = lowr["Ea"] * eF
            if "troe" in x:
                kind[r] = KIND_TROE
                tr = x["troe"]
                troe[r] = [tr["alpha"], tr["T3"], tr["T1"], tr.get("T2", 0.0)]
            else:
                kind[r] = KIND_LINDEMANN
        else:
            raise ValueError(f"unknown reaction type {t}")
        b[r] = rate["b"]
        Ea[r] = rate["Ea"] * eF
        for s, v in x.get("efficiencies", {}).items():
            eff[r, names.index(s)] = float(v)
    m = OracleMechanism(doc["name"], names, elements, W, comp, T_range, lo, hi, nu_f, nu_r,
                        A, b, Ea, kind, rev, eff, A0, b0, Ea0, troe)
    check_balance(m)
    return m


def check_balance(m: OracleMechanism, tol=1e-12):
    """S:28 / S:82: sum_k nu_kr W_k = 0 (relative 1e-12) and exact element balance per row."""
    nu = m.nu_r - m.nu_f
    for r in range(m.nr):
        dm = float(nu[r] @ m.W)
        gross = float(np.abs(nu[r]) @ m.W)
        if abs(dm) > tol * gross:
            raise ValueError(f"reaction {r}: mass imbalance {dm}")
        if np.any(nu[r] @ m.comp != 0):
            raise ValueError(f"reaction {r}: element imbalance")

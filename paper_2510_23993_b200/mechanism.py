"""Product-side mechanism loader: YAML file in mech/ -> the host tables of `chem_mech_desc`
(include/chem.h) in SI-molar units.

Independent of oracle/mechanism.py (the two share only the data file).  The library re-validates
everything in `chem_init` (mass/element balance, ranges, types); this module only parses and
converts units.  Unit conventions follow the file header: rate constants of an elementary row of
reaction order m are in (length^3/mol)^(m-1)/s, a three-body row counts [M] in its order, a falloff
row's low-pressure limit k0 multiplies [M] (PAPER.md P:78 cites the mechanism; CHEMKIN semantics).
"""
from __future__ import annotations

import dataclasses
import pathlib

import numpy as np
import yaml

R_UNIVERSAL = 8.314462618
P_STANDARD = 101325.0

TYPE_ELEMENTARY = 0
TYPE_THREE_BODY = 1
TYPE_LINDEMANN = 2
TYPE_TROE = 3

MECH_DIR = pathlib.Path(__file__).resolve().parent.parent / "mech"


@dataclasses.dataclass
class MechTables:
    name: str
    species: list
    elements: list
    W: np.ndarray          # [ns]
    nasa_lo: np.ndarray    # [ns, 7]
    nasa_hi: np.ndarray    # [ns, 7]
    T_range: np.ndarray    # [ns, 3]
    elem: np.ndarray       # [ns, ne] int32
    nu_f: np.ndarray       # [nr, ns] float64
    nu_r: np.ndarray       # [nr, ns]
    A: np.ndarray
    b: np.ndarray
    Ea: np.ndarray         # J/mol
    type: np.ndarray       # [nr] int32
    reversible: np.ndarray  # [nr] int32
    eff: np.ndarray        # [nr, ns]
    A0: np.ndarray
    b0: np.ndarray
    Ea0: np.ndarray
    troe: np.ndarray       # [nr, 4]  alpha, T***, T*, T** (0 = absent)

    @property
    def ns(self):
        return len(self.species)

    @property
    def nr(self):
        return len(self.A)

    @property
    def ne(self):
        return len(self.elements)


def find(name_or_path) -> pathlib.Path:
    p = pathlib.Path(name_or_path)
    return p if p.suffix in (".yaml", ".yml") and p.exists() else MECH_DIR / f"{name_or_path}.yaml"


def load(name_or_path) -> MechTables:
    path = find(name_or_path)
    doc = yaml.safe_load(path.read_text())
    u = doc.get("units", {})
    conc_unit = {"m": 1.0, "cm": 1e-6}[u.get("length", "m")]            # length^3 -> m^3
    e_unit = {"J/mol": 1.0, "cal/mol": 4.184, "kcal/mol": 4184.0}[u.get("activation-energy", "J/mol")]
    weights = doc["atomic_weights"]
    elements = list(weights)
    names = [sp["name"] for sp in doc["species"]]
    ns, ne = len(names), len(elements)
    elem = np.zeros((ns, ne), dtype=np.int32)
    for i, sp in enumerate(doc["species"]):
        for el, n in sp["composition"].items():
            elem[i, elements.index(el)] = n
    W = np.array([sum(weights[el] * n for el, n in sp["composition"].items()) for sp in doc["species"]]) / 1000.0
    nasa_lo = np.array([sp["low"] for sp in doc["species"]], dtype=np.float64)
    nasa_hi = np.array([sp["high"] for sp in doc["species"]], dtype=np.float64)
    T_range = np.array([sp["T_range"] for sp in doc["species"]], dtype=np.float64)

    rows = doc["reactions"]
    nr = len(rows)
    nu_f = np.zeros((nr, ns))
    nu_r = np.zeros((nr, ns))
    A = np.zeros(nr); b = np.zeros(nr); Ea = np.zeros(nr)
    A0 = np.zeros(nr); b0 = np.zeros(nr); Ea0 = np.zeros(nr)
    typ = np.zeros(nr, dtype=np.int32)
    rev = np.zeros(nr, dtype=np.int32)
    eff = np.ones((nr, ns))
    troe = np.zeros((nr, 4))
    for r, row in enumerate(rows):
        for s, v in row["reactants"].items():
            nu_f[r, names.index(s)] = v
        for s, v in row["products"].items():
            nu_r[r, names.index(s)] = v
        m = nu_f[r].sum()
        kind = row.get("type", "elementary")
        rev[r] = int(bool(row.get("reversible", True)))
        if kind == "falloff":
            hi, lo = row["high"], row["low"]
            A[r], b[r], Ea[r] = hi["A"] * conc_unit ** (m - 1), hi["b"], hi["Ea"] * e_unit
            A0[r], b0[r], Ea0[r] = lo["A"] * conc_unit ** m, lo["b"], lo["Ea"] * e_unit
            if "troe" in row:
                t = row["troe"]
                typ[r] = TYPE_TROE
                troe[r] = (t["alpha"], t["T3"], t["T1"], t.get("T2", 0.0))
            else:
                typ[r] = TYPE_LINDEMANN
        else:
            k = row["rate"]
            order_extra = 1 if kind == "three-body" else 0
            typ[r] = TYPE_THREE_BODY if kind == "three-body" else TYPE_ELEMENTARY
            A[r], b[r], Ea[r] = k["A"] * conc_unit ** (m - 1 + order_extra), k["b"], k["Ea"] * e_unit
        for s, v in row.get("efficiencies", {}).items():
            eff[r, names.index(s)] = v
    return MechTables(doc["name"], names, elements, W, nasa_lo, nasa_hi, T_range, elem, nu_f, nu_r,
                      A, b, Ea, typ, rev, eff, A0, b0, Ea0, troe)

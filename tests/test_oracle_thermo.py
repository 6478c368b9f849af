"""Pins for the oracle's thermo and temperature recovery (SURVEY.md §8(c) "Thermo"; SPEC.md
S:54-79).  Every expectation is fixed by something other than the oracle: textbook
JANAF values, continuity of the NASA fits, d u/dT = c_v, linear mixing, and the closed-form
one-step Newton for a constant-cv gas."""
import os

import numpy as np
import pytest

from oracle import Oracle, load_mechanism

GOLD = os.path.join(os.path.dirname(__file__), "golden")
R = 8.314462618


def _rows(name):
    out = []
    for line in open(os.path.join(GOLD, name)):
        if line.strip() and not line.startswith("#"):
            out.append(line.split())
    return out


def test_janaf_298(oracle_h2):
    o = oracle_h2
    cp, h, s = o.thermo(298.15)
    for sp, dh, tdh, S, tS, c, tc in _rows("thermo_298_janaf.txt"):
        k = o.m.species.index(sp)
        assert abs(h[k] / 1e3 - float(dh)) <= float(tdh), (sp, h[k])
        # 1 bar vs 1 atm standard state: S(1 atm) = S(1 bar) - R ln(1.01325)
        assert abs(s[k] - (float(S) - R * np.log(1.01325))) <= float(tS) + 0.12, (sp, s[k])
        assert abs(cp[k] - float(c)) <= float(tc), (sp, cp[k])


def test_janaf_cp_2000K(oracle_h2):
    cp, _, _ = oracle_h2.thermo(2000.0)
    for sp, c, tol in _rows("cp_2000K_janaf.txt"):
        k = oracle_h2.m.species.index(sp)
        assert abs(cp[k] / float(c) - 1) < float(tol), (sp, cp[k])


def test_nasa_continuity_at_Tmid(oracle_h2):
    """The two NASA-7 ranges are fitted to join at T_mid; a mistyped coefficient breaks this."""
    Tm = 1000.0
    a = oracle_h2.thermo(Tm * (1 - 1e-12))
    b = oracle_h2.thermo(Tm * (1 + 1e-12))
    assert np.max(np.abs(a[0] - b[0]) / np.abs(b[0])) < 1e-5          # cp
    assert np.max(np.abs(a[1] - b[1])) < 1e-5 * R * Tm * 10              # h  (J/mol)
    assert np.max(np.abs(a[2] - b[2]) / np.abs(b[2])) < 1e-5          # s


def test_cv_is_du_dT(oracle_h2):
    """d u/dT = c_v (central finite difference)."""
    rng = np.random.default_rng(1)
    for _ in range(20):
        Y = rng.dirichlet(np.ones(9))
        T = rng.uniform(400, 2900)
        if abs(T - 1000) < 5:
            continue
        dT = 1e-3
        fd = (oracle_h2.energy(T + dT, Y) - oracle_h2.energy(T - dT, Y)) / (2 * dT)
        assert abs(fd / oracle_h2.cv(T, Y) - 1) < 1e-8


def test_u_strictly_increasing(oracle_h2):
    rng = np.random.default_rng(2)
    Ts = np.linspace(250, 3400, 400)
    for _ in range(10):
        Y = rng.dirichlet(np.ones(9))
        u = np.array([oracle_h2.energy(T, Y) for T in Ts])
        assert np.all(np.diff(u) > 0)


def test_newton_round_trip(oracle_h2):
    """T -> u -> Newton recovers T (here within 1e-9 K)."""
    rng = np.random.default_rng(3)
    for _ in range(100):
        Y = rng.dirichlet(0.5 * np.ones(9))
        T = rng.uniform(300, 3000)
        e = oracle_h2.energy(T, Y)
        Tn, it = oracle_h2.newton_T(e, Y, T_guess=rng.uniform(300, 3000))
        assert it > 0 and abs(Tn - T) < 1e-9


def test_newton_one_step_constant_cv():
    """for a constant-cv gas u is linear in T, so the first Newton update is exact."""
    o = Oracle("toy_a_to_b")
    Y = np.array([0.3, 0.7])
    e = o.energy(1500.0, Y)
    cv = o.cv(1500.0, Y)
    assert abs(cv - 2.5 * R / 0.028) < 1e-9 * cv          # cp = 3.5 R  ->  cv = 2.5 R / W
    Tn, it = o.newton_T(e, Y, 400.0)
    assert it <= 2 and abs(Tn - 1500.0) < 1e-10


def test_mixture_cv_linear():
    """mixture cv is mass-fraction weighted (700/900 analogue with the toy gases)."""
    o = Oracle("toy_2a_to_b")
    cvA = 1.5 * R / 0.020
    cvB = 3.0 * R / 0.040
    assert abs(o.cv(900.0, np.array([0.5, 0.5])) - 0.5 * (cvA + cvB)) < 1e-10 * cvA


def test_mechanism_balance_and_rejects_imbalance(tmp_path):
    """the loader enforces per-reaction mass and element balance."""
    m = load_mechanism("h2air_li2004")
    nu = m.nu_r - m.nu_f
    assert m.ns == 9 and m.nr == 21
    assert np.all(nu @ m.comp == 0)
    assert np.max(np.abs(nu @ m.W)) < 1e-15
    src = open(os.path.join(os.path.dirname(GOLD), "..", "mech", "toy_a_to_b.yaml")).read()
    bad = src.replace("products: {B: 1}", "products: {B: 2}")
    p = tmp_path / "bad.yaml"
    p.write_text(bad)
    with pytest.raises(ValueError):
        load_mechanism(str(p))

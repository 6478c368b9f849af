"""NEXT-3: the larger published mechanism mech/gri30_hon.yaml
(GRI-Mech 3.0 H/O/N/Ar subset, 14 species, 41 rows) pinned on the oracle side the way the 9-species
one is: JANAF 298 K values of the added species, NASA continuity at T_mid, the per-reaction loop ==
the independent numpy matrix form, chain-branching rates against Baulch 2005, both loaders equal, and
relaxation (with thermal NO) to an independent element-potential equilibrium in detailed balance."""
import os

import numpy as np
import pytest

from oracle import Oracle
from oracle import mechanism as omech
from tests.pins.ignition import equilibrium_uv, rho_of
from tests.pins.matrix_rates import gross, matrix_rates

GOLD = os.path.join(os.path.dirname(__file__), "golden")
R = 8.314462618
NA = 6.02214076e23


@pytest.fixture(scope="module")
def gri():
    return Oracle("gri30_hon")


def test_shape(gri):
    m = gri.m
    assert (m.ns, m.nr) == (14, 41)
    net = m.nu_r - m.nu_f
    assert [m.species[k] for k in range(m.ns) if not np.any(net[:, k])] == ["AR"]   # 13 reacting + T


def test_janaf_298_added_species(gri):
    cp, h, s = gri.thermo(298.15)
    for line in open(os.path.join(GOLD, "thermo_298_janaf_nox.txt")):
        if not line.strip() or line.startswith("#"):
            continue
        sp, dh, tdh, S, tS, c, tc = line.split()
        k = gri.m.species.index(sp)
        assert abs(h[k] / 1e3 - float(dh)) <= float(tdh), (sp, h[k])
        assert abs(s[k] - (float(S) - R * np.log(1.01325))) <= float(tS) + 0.12, (sp, s[k])
        assert abs(cp[k] - float(c)) <= float(tc), (sp, cp[k])


def test_nasa_continuity(gri):
    m = gri.m
    lo, hi = gri.thermo(999.999999), gri.thermo(1000.000001)
    for a, b in zip(lo, hi):
        assert np.max(np.abs(a / b - 1)) < 1e-6


def _states(m, n, seed):
    rng = np.random.default_rng(seed)
    T = rng.uniform(600.0, 3000.0, n)
    p = 101325.0 * 10 ** rng.uniform(-1, 2, n)
    Y = rng.dirichlet(np.full(m.ns, 0.5), n)
    Y[rng.random(Y.shape) < 0.2] = 0.0
    Y /= Y.sum(1, keepdims=True)
    rho = p / (R * T * (Y / m.W).sum(1))
    return rho, T, Y


def test_loop_equals_matrix_form(gri):
    m = gri.m
    rho, T, Y = _states(m, 300, 5)
    w_mat, qf_mat, qr_mat = matrix_rates(m, rho, T, Y)
    G = gross(m, qf_mat, qr_mat)
    for i in range(len(rho)):
        w, qf, qr = gri.rates(rho[i], T[i], Y[i])
        assert np.all(np.abs(w - w_mat[i]) <= 1e-12 * G[i] + 1e-300), i


def test_chain_rates_vs_baulch_2005(gri):
    m = gri.m
    sp = m.species.index

    def row(reac, prod):
        for r in range(m.nr):
            if set(np.nonzero(m.nu_f[r])[0]) == {sp(x) for x in reac} and \
                    set(np.nonzero(m.nu_r[r])[0]) == {sp(x) for x in prod}:
                return r
        raise KeyError(reac)
    lit = {(("H", "O2"), ("O", "OH")): lambda T: 3.43e-10 * T ** -0.097 * np.exp(-7560.0 / T),
           (("O", "H2"), ("H", "OH")): lambda T: 8.5e-20 * T ** 2.67 * np.exp(-3160.0 / T),
           (("OH", "H2"), ("H", "H2O")): lambda T: 1.55e-12 * (T / 298.0) ** 1.6 * np.exp(-1660.0 / T)}
    for (reac, prod), f in lit.items():
        r = row(reac, prod)
        for T in (1000.0, 1500.0, 2000.0, 2500.0):
            k = m.A[r] * T ** m.b[r] * np.exp(-m.Ea[r] / (R * T)) * 1e6 / NA
            assert 1 / 1.5 < k / f(T) < 1.5, (reac, T, k / f(T))


def test_loaders_agree():
    from paper_2510_23993_b200 import mechanism as pmech
    o, p = omech.load("gri30_hon"), pmech.load("gri30_hon")
    for a in ("A", "b", "Ea", "A0", "b0", "Ea0", "W", "troe", "eff"):
        np.testing.assert_allclose(np.asarray(getattr(p, a), float), np.asarray(getattr(o, a), float),
                                   rtol=1e-14, atol=0)


def _air_fuel(m):
    X = np.zeros(m.ns)
    X[m.species.index("H2")] = 2.0
    X[m.species.index("O2")] = 1.0
    X[m.species.index("N2")] = 3.714
    X[m.species.index("AR")] = 0.046          # air O2:N2:Ar = 21:78:1 by moles
    Y = X * m.W
    return Y / Y.sum()


def test_relaxation_to_equilibrium_with_thermal_no(gri):
    """1 s from stoichiometric H2-air (with Ar) at 1500 K, 1 atm: the long-time oracle state equals an
    independent constant-(u, v) element-potential equilibrium (thermo + elements only, 4 elements),
    including NO (thermal NO at ~2400 K), and every reversible row is in detailed balance."""
    m = gri.m
    Y0 = _air_fuel(m)
    T0 = 1500.0
    rho = rho_of(m, 101325.0, T0, Y0)
    e = gri.energy(T0, Y0)
    y, _ = gri.integrate_state(rho, np.r_[Y0, T0], 1.0)
    Teq, Yeq, res = equilibrium_uv(m, rho, e, Y0)
    assert res < 1e-12
    assert abs(y[-1] / Teq - 1) < 1e-6
    mask = Yeq > 1e-10
    assert Yeq[m.species.index("NO")] > 1e-3         # thermal NO is formed at equilibrium
    assert np.max(np.abs(y[:-1][mask] / Yeq[mask] - 1)) < 1e-6
    _, qf, qr = gri.rates(rho, y[-1], y[:-1])
    rev = (m.reversible == 1) & (qf > 1e-200)
    assert np.max(np.abs(np.log(qf[rev]) - np.log(qr[rev]))) < 1e-6

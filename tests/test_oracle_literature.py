"""Soft literature pins of the transcribed Li-2004 kinetics (SURVEY.md §8(c) last
row: "transcription errors in A, b, Ea are caught only by a soft comparison to literature values").

No Cantera offline and PAPER.md prints no rate or delay values (only R^2), so the constants in
mech/h2air_li2004.yaml, as converted to SI by each loader, are compared with INDEPENDENT literature
evaluations of the same elementary rates and with a shock-tube induction-time correlation.  The
bars are soft (factors of 1.5-3) because the sources are different evaluations; what they catch is
a mistyped exponent, a wrong unit conversion (cm^3 -> m^3 per concentration order, cal -> J) or a
swapped row, each of which moves a rate by orders of magnitude.

Sources (values as published, cm^3 molecule^-1 s^-1 unless stated):
  [B05] D. L. Baulch et al., J. Phys. Chem. Ref. Data 34 (2005) 757:
        H + O2 -> OH + O   k = 3.43e-10 T^-0.097 exp(-7560/T)          (1000-3500 K)
        O + H2 -> OH + H   k = 8.5e-20 T^2.67 exp(-3160/T)             (300-2500 K)
        OH + H2 -> H + H2O k = 1.55e-12 (T/298)^1.6 exp(-1660/T)       (250-2500 K)
  [JPL] JPL/NASA Evaluation No. 17 (2011): H + O2 + M -> HO2 + M, low-pressure limit in air,
        k0 = 4.4e-32 (T/300)^-1.3 cm^6 molecule^-2 s^-1.
  [SK]  D. Schott, J. L. Kinsey, J. Chem. Phys. 29 (1958) 1177: H2-O2 induction times behind shock
        waves, log10(tau [O2]) = -10.7 + 3960/T  (tau in s, [O2] in mol/L; OH-onset induction time in
        Ar-diluted mixtures, hence only a factor-3 bar on the level and 25 % on the slope here, where
        tau is the time of max dT/dt in air, SURVEY reading 16).
  [SW]  A. L. Sanchez, F. A. Williams, Prog. Energy Combust. Sci. 41 (2014) 1: the crossover
        temperature 2 k1 = k9 [M] of H2-air at 1 atm lies near 950-1000 K (bar: 900-1050 K).
"""
import numpy as np
import pytest

from oracle import mechanism as omech

NA = 6.02214076e23
R = 8.314462618


def _k(m, r, T):
    """Forward rate constant of row r from the LOADED (SI) tables: k = A T^b exp(-Ea/RT)."""
    return m.A[r] * T ** m.b[r] * np.exp(-m.Ea[r] / (R * T))


def _k0(m, r, T):
    return m.A0[r] * T ** m.b0[r] * np.exp(-m.Ea0[r] / (R * T))


def _row(m, eq):
    idx = [i for i in range(m.nr) if _eq(m, i) == eq]
    assert len(idx) == 1, eq
    return idx[0]


def _eq(m, r):
    side = lambda v: " + ".join(sorted(sum(([m.species[k]] * int(v[k]) for k in range(m.ns)), [])))  # noqa: E731
    return f"{side(m.nu_f[r])} => {side(m.nu_r[r])}"


def _si_to_molecule(k_si, order=2):
    """m^3/(mol s) (order 2) or m^6/(mol^2 s) (order 3) -> cm^3/molecule/s or cm^6/molecule^2/s."""
    return k_si * (1e6 / NA) ** (order - 1)


@pytest.fixture(scope="module", params=["oracle", "product"])
def mech(request):
    """Both loaders' SI tables (each converts the CHEMKIN units independently)."""
    if request.param == "oracle":
        return omech.load("h2air_li2004")
    from paper_2510_23993_b200 import mechanism as pmech
    return pmech.load("h2air_li2004")


@pytest.mark.parametrize("eq,lit,T_range", [
    ("H + O2 => O + OH", lambda T: 3.43e-10 * T ** -0.097 * np.exp(-7560.0 / T), (1000.0, 2500.0)),
    ("H2 + O => H + OH", lambda T: 8.5e-20 * T ** 2.67 * np.exp(-3160.0 / T), (500.0, 2500.0)),
    ("H2 + OH => H + H2O", lambda T: 1.55e-12 * (T / 298.0) ** 1.6 * np.exp(-1660.0 / T), (500.0, 2500.0)),
])
def test_chain_rates_vs_baulch_2005(mech, eq, lit, T_range):
    """[B05]: the three chain-branching / propagation rates within a factor 1.5 over their ranges."""
    m = mech
    r = _row(m, eq)
    for T in np.linspace(*T_range, 7):
        ratio = _si_to_molecule(_k(m, r, T)) / lit(T)
        assert 1 / 1.5 < ratio < 1.5, (eq, T, ratio)


def test_h_o2_m_low_pressure_limit_vs_jpl(mech):
    """[JPL]: k0 of H + O2 (+M) -> HO2 (+M) (falloff row; unit conversion cm^6/mol^2 -> m^6/mol^2)
    within a factor 1.5 at 300-1000 K for N2 (efficiency 1 in Li 2004)."""
    m = mech
    r = _row(m, "H + O2 => HO2")
    kind = getattr(m, "kind", None)
    kind = m.type if kind is None else kind
    assert int(kind[r]) == 3                      # Troe falloff row
    for T in (300.0, 500.0, 1000.0):
        ratio = _si_to_molecule(_k0(m, r, T), order=3) / (4.4e-32 * (T / 300.0) ** -1.3)
        assert 1 / 1.5 < ratio < 1.5, (T, ratio)


def test_crossover_temperature_1atm(mech):
    """[SW]: 2 k1 = k9 [M] (branching vs the HO2-forming termination) at 1 atm, stoichiometric
    H2-air (efficiencies of the row applied), lies between 900 and 1050 K."""
    m = mech
    r1 = _row(m, "H + O2 => O + OH")
    r9 = _row(m, "H + O2 => HO2")
    X = np.zeros(m.ns)
    X[m.species.index("H2")] = 2.0
    X[m.species.index("O2")] = 1.0
    X[m.species.index("N2")] = 3.76
    X /= X.sum()

    def g(T):
        c = 101325.0 / (R * T) * X
        M = float(m.eff[r9] @ c)
        kinf = _k(m, r9, T)
        Pr = _k0(m, r9, T) * M / kinf
        alpha = m.troe[r9][0]                     # Li 2004: T*** = 1e-30, T* = 1e30 -> Fcent = alpha
        Fc = alpha
        cc = -0.4 - 0.67 * np.log10(Fc)
        nn = 0.75 - 1.27 * np.log10(Fc)
        f1 = (np.log10(Pr) + cc) / (nn - 0.14 * (np.log10(Pr) + cc))
        F = 10.0 ** (np.log10(Fc) / (1.0 + f1 * f1))
        k9 = kinf * Pr / (1.0 + Pr) * F           # effective bimolecular rate (M folded in)
        return 2.0 * _k(m, r1, T) - k9
    from scipy.optimize import brentq
    Tc = brentq(g, 600.0, 1500.0)
    assert 900.0 < Tc < 1050.0, Tc


def test_ignition_delay_vs_schott_kinsey(oracle_h2):
    """[SK]: tau_ign of stoichiometric H2-air at 1 atm, 1500-2500 K (the conditions of P:456) against
    log10(tau [O2]) = -10.7 + 3960/T: level within a factor 3 at every T0, apparent activation
    temperature (slope of log10(tau [O2]) vs 1/T0) within 25 %."""
    from tests.pins.ignition import fresh_Y, ignition_delay, rho_of
    o = oracle_h2
    m = o.m
    Y0 = fresh_Y(m)
    Ts = np.array([1500.0, 1750.0, 2000.0, 2250.0, 2500.0])
    xo2 = (Y0 / m.W)[m.species.index("O2")] / np.sum(Y0 / m.W)
    lt = []
    for T0 in Ts:
        tau = ignition_delay(o, rho_of(m, 101325.0, T0, Y0), np.r_[Y0, T0], 3e-3)
        o2 = xo2 * 101325.0 / (R * T0) * 1e-3        # mol/L
        lt.append(np.log10(tau * o2))
    lt = np.array(lt)
    sk = -10.7 + 3960.0 / Ts
    assert np.all(np.abs(lt - sk) < np.log10(3.0)), (lt, sk)
    slope = np.polyfit(1.0 / Ts, lt, 1)[0]
    assert abs(slope / 3960.0 - 1) < 0.25, slope


def test_loaders_agree(mech):
    """The two independent loaders produce the same SI tables (rows in file order)."""
    o = omech.load("h2air_li2004")
    m = mech
    for a in ("A", "b", "Ea", "A0", "b0", "Ea0", "W"):
        np.testing.assert_allclose(np.asarray(getattr(m, a), float), np.asarray(getattr(o, a), float),
                                   rtol=1e-14, atol=0)
    np.testing.assert_array_equal(np.asarray(m.nu_f, float), np.asarray(o.nu_f, float))
    np.testing.assert_allclose(np.asarray(m.eff, float), o.eff, rtol=0, atol=0)

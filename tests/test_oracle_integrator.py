"""Pins for the oracle's integrator and cell loop (SURVEY.md §8(c) "Integrator accuracy",
"Oracle integrator, library check", "Linear invariants", "K_c and thermo" (equilibrium),
"Trends", "Cold cells").  Expected values come from closed forms, scipy's independent
Radau/BDF, an independent Gibbs/element-potential equilibrium solve, and the physics."""
import numpy as np
import pytest
from scipy.integrate import solve_ivp

from oracle import Oracle
from tests.pins.ignition import equilibrium_uv, fresh_Y, ignition_delay, rho_of

R = 8.314462618
P_ATM = 101325.0


# ---------------------------------------------------------------- closed forms (toy mechanisms)

def test_closed_form_a_to_b():
    """A->B: Y_A(t) = Y_A0 exp(-k t), isothermal by construction.  Oracle at its
    reference rtol 1e-12."""
    o = Oracle("toy_a_to_b")
    k = 1e3
    for t in (1e-4, 1e-3, 5e-3):
        y, _ = o.integrate_state(1.0, np.array([0.8, 0.2, 600.0]), t, rtol=1e-12, atolY=1e-20, atolT=1e-9)
        exact = 0.8 * np.exp(-k * t)
        assert abs(y[0] / exact - 1) < 1e-9
        assert abs(y[1] - (1.0 - exact)) < 1e-9
        assert abs(y[2] - 600.0) < 1e-9


def test_closed_form_a_eq_b():
    """A<=>B with K_c = 1: c_A = cbar + (c_A0 - cbar) exp(-2 k t)."""
    o = Oracle("toy_a_eq_b")
    k = 1e3
    for t in (2e-4, 1e-3, 4e-3):
        y, _ = o.integrate_state(2.0, np.array([0.9, 0.1, 800.0]), t, rtol=1e-12, atolY=1e-20, atolT=1e-9)
        exact = 0.5 + (0.9 - 0.5) * np.exp(-2 * k * t)
        assert abs(y[0] / exact - 1) < 1e-9


def test_closed_form_2a_to_b():
    """2A->B: c_A = c0/(1 + 2 k c0 t)."""
    o = Oracle("toy_2a_to_b")
    k, rho, WA = 10.0, 1.0, 0.020
    c0 = rho * 1.0 / WA
    for t in (1e-4, 1e-3, 1e-2):
        y, _ = o.integrate_state(rho, np.array([1.0, 0.0, 900.0]), t, rtol=1e-12, atolY=1e-20, atolT=1e-9)
        exact = c0 / (1 + 2 * k * c0 * t)
        assert abs(y[0] * rho / WA / exact - 1) < 1e-9
        assert abs(y[2] - 900.0) < 1e-8


def _cgs_state(o):
    from tests.pins import cgs_toy as ct
    rho = ct.rho_at_troe_centre()
    Y = np.zeros(o.m.ns)
    for k, v in ct.Y0.items():
        Y[o.m.species.index(k)] = v
    return ct, rho, Y


def test_cgs_toy_rates_closed_form():
    """the oracle loader's cm/cal conversion of three-body, Lindemann, Troe and
    second-order rows, pinned by the hand-converted SI closed forms of tests/pins/cgs_toy.py at t = 0:
    Omega_A1 = -lam1 c_A1, Omega_A2 = -lam2 c_A2, Omega_A3 = -lam3 c_A3, Omega_A4 = -2 k4 c_A4^2."""
    o = Oracle("toy_cgs_falloff")
    ct, rho, Y = _cgs_state(o)
    lam1, lam2, lam3, k4 = ct.decay_rates(rho)
    w, _, _ = o.rates(rho, ct.T, Y)
    sp = o.m.species.index
    c = rho * Y / ct.W
    exp = {"A1": -lam1 * c[sp("A1")], "A2": -lam2 * c[sp("A2")], "A3": -lam3 * c[sp("A3")],
           "A4": -2.0 * k4 * c[sp("A4")] ** 2}
    for k, v in exp.items():
        assert abs(w[sp(k)] / v - 1) < 1e-12, (k, w[sp(k)], v)
    assert abs(w[sp("B4")] / (-0.5 * exp["A4"]) - 1) < 1e-12
    assert w[sp("N")] == 0.0


def test_cgs_toy_integrated_closed_form():
    """The same pins through the oracle integrator: Y_Ai(t) against the closed forms over one dt at
    T = 1000 K (isothermal by construction), rtol 1e-12 -> 1e-9 relative."""
    o = Oracle("toy_cgs_falloff")
    ct, rho, Y = _cgs_state(o)
    sp = o.m.species.index
    for t in (2e-6, 1e-5):
        y, _ = o.integrate_state(rho, np.r_[Y, ct.T], t, rtol=1e-12, atolY=1e-24, atolT=1e-9)
        ex = ct.exact_Y(rho, t)
        for name, v in zip(("A1", "A2", "A3", "A4"), ex):
            assert abs(y[sp(name)] / v - 1) < 1e-9, (name, t, y[sp(name)], v)
        assert abs(y[-1] - ct.T) < 1e-8


# ---------------------------------------------------------------- scipy library check

def _cases(o):
    m = o.m
    Y0 = fresh_Y(m)
    cases = []
    for T0, dt in ((1000.0, 1e-7), (1200.0, 1e-7), (1500.0, 1e-7), (1200.0, 1e-4), (1100.0, 1e-4)):
        rho = rho_of(m, P_ATM, T0, Y0)
        cases.append((rho, np.r_[Y0, T0], dt))
    # radical-rich mid-induction state (cfg1b-like): advance 1200 K fresh gas to 0.9 tau
    rho = rho_of(m, P_ATM, 1200.0, Y0)
    ymid, _ = o.integrate_state(rho, np.r_[Y0, 1200.0], 0.9 * 4.3999e-5)
    cases.append((rho, ymid, 1e-7))
    cases.append((rho, ymid, 1e-5))
    return cases


@pytest.mark.parametrize("method", ["Radau", "BDF"])
def test_oracle_vs_scipy(oracle_h2, method):
    o = oracle_h2
    for rho, y0, dt in _cases(o):
        y, _ = o.integrate_state(rho, y0, dt, rtol=1e-12, atolY=1e-24, atolT=1e-9)
        atol = np.r_[np.full(o.ns, 1e-24), 1e-9]
        sol = solve_ivp(lambda t, y: o.rhs(rho, y), (0.0, dt), y0, method=method, rtol=1e-12, atol=atol,
                        jac=lambda t, y: o.jac(rho, y))
        assert sol.success
        ys = sol.y[:, -1]
        mask = np.r_[ys[:-1] > 1e-12, True]
        rel = np.abs(y[mask] / ys[mask] - 1)
        assert rel.max() < 1e-8, (dt, rel.max())


# ---------------------------------------------------------------- invariants and gate

def _cfg1_like(o, n=64, seed=5):
    m = o.m
    Y0 = fresh_Y(m)
    T0 = np.linspace(900.0, 1500.0, n)
    rho = np.array([rho_of(m, P_ATM, t, Y0) for t in T0])
    Y = np.tile(Y0, (n, 1))
    e = np.array([o.energy(t, Y0) for t in T0])
    return rho, e, T0, Y


def test_linear_invariants(oracle_h2):
    """sum Y - 1, element moles, rho, and e(T_out, Y_out) = e_in."""
    o = oracle_h2
    m = o.m
    rho, e, T0, Y = _cfg1_like(o, 48)
    out = o.integrate_cells(rho, e, T0, Y, 1e-4, rtol=1e-10, atolY=1e-20, atolT=1e-6)
    assert np.all(out["status"] == 0)
    Yo = out["Y"]
    assert np.max(np.abs(Yo.sum(1) - 1)) < 1e-13
    el0 = (Y / m.W) @ m.comp
    el1 = (Yo / m.W) @ m.comp
    assert np.max(np.abs(el1 / el0 - 1)) < 1e-12
    e_out = np.array([o.energy(t, y) for t, y in zip(out["T"], Yo)])
    assert np.max(np.abs(e_out / e - 1)) < 1e-12
    # the integrated T tracks the Newton T (energy drift of Eq. 6 integration)
    assert np.max(np.abs(out["T_int"] / out["T"] - 1)) < 1e-6


def test_gate_cold_and_solid_untouched(oracle_h2):
    """T < T_min or solid -> state bitwise untouched."""
    o = oracle_h2
    rho, e, T0, Y = _cfg1_like(o, 16)
    T0 = T0.copy()
    T0[:4] = 300.0
    solid = np.zeros(16, dtype=np.uint8)
    solid[10] = 1
    out = o.integrate_cells(rho, e, T0, Y, 1e-6, rtol=1e-8, T_min=500.0, solid=solid)
    for i in list(range(4)) + [10]:
        assert out["status"][i] == 1
        assert out["T"][i] == T0[i] and np.array_equal(out["Y"][i], Y[i])
    assert np.all(out["status"][4:10] == 0)


def test_self_convergence(oracle_h2):
    """rtol 1e-12 and 1e-13 agree to 1e-9 relative (Y > 1e-12)."""
    o = oracle_h2
    for rho, y0, dt in _cases(o):
        a, _ = o.integrate_state(rho, y0, dt, rtol=1e-12)
        b, _ = o.integrate_state(rho, y0, dt, rtol=1e-13)
        mask = np.r_[b[:-1] > 1e-12, True]
        assert np.max(np.abs(a[mask] / b[mask] - 1)) < 1e-9


# ---------------------------------------------------------------- equilibrium and trends

def test_relaxation_to_equilibrium(oracle_h2):
    """BJ:5 'relaxation to equilibrium': 1 s from phi=1 at 1500 K, 1 atm reaches the
    constant-(u,v) equilibrium of an independent element-potential solve (thermo only), and
    every reversible row is in detailed balance (|ln qf - ln qr| <= 1e-6)."""
    o = oracle_h2
    m = o.m
    Y0 = fresh_Y(m)
    T0 = 1500.0
    rho = rho_of(m, P_ATM, T0, Y0)
    e = o.energy(T0, Y0)
    y, _ = o.integrate_state(rho, np.r_[Y0, T0], 1.0)
    Teq, Yeq, res = equilibrium_uv(m, rho, e, Y0)
    assert res < 1e-12
    assert abs(y[-1] / Teq - 1) < 1e-6
    mask = Yeq > 1e-10
    assert np.max(np.abs(y[:-1][mask] / Yeq[mask] - 1)) < 1e-6
    _, qf, qr = o.rates(rho, y[-1], y[:-1])
    rev = m.reversible == 1
    assert np.max(np.abs(np.log(qf[rev]) - np.log(qr[rev]))) < 1e-6


def test_ignition_delay_trends(oracle_h2):
    """P:456 / S:604: tau_ign strictly decreasing in T0 (cfg1 range 1000-1500 K and the
    paper's 1500-2500 K) and ln tau vs 1/T0 with R^2 > 0.9 on 1500-2500 K."""
    o = oracle_h2
    m = o.m
    Y0 = fresh_Y(m)
    T_a = [1000.0, 1100.0, 1200.0, 1300.0, 1400.0, 1500.0]
    T_b = [1500.0, 1750.0, 2000.0, 2250.0, 2500.0]
    taus = {}
    for T0 in sorted(set(T_a + T_b)):
        taus[T0] = ignition_delay(o, rho_of(m, P_ATM, T0, Y0), np.r_[Y0, T0], 3e-3)
    for Ts in (T_a, T_b):
        t = [taus[x] for x in Ts]
        assert all(a > b for a, b in zip(t, t[1:])), t
    x = 1.0 / np.array(T_b)
    yv = np.log([taus[T] for T in T_b])
    A = np.vstack([x, np.ones_like(x)]).T
    coef, *_ = np.linalg.lstsq(A, yv, rcond=None)
    r2 = 1 - np.sum((yv - A @ coef) ** 2) / np.sum((yv - yv.mean()) ** 2)
    assert r2 > 0.9
    assert coef[0] > 0          # Arrhenius: tau grows with 1/T


def test_ignition_helper_refuses_non_igniting_mixture(oracle_h2):
    """a mixture with no interior max of dT/dt (cold, 600 K) must raise instead
    of returning an extrapolated (negative) tau; the BDF refuses a negative interval (rc -5)."""
    from oracle.ignition import NoIgnition
    o = oracle_h2
    m = o.m
    Y0 = fresh_Y(m)
    with pytest.raises(NoIgnition):
        ignition_delay(o, rho_of(m, P_ATM, 600.0, Y0), np.r_[Y0, 600.0], 1e-3, t_max=4e-3)
    with pytest.raises(RuntimeError, match="rc=-5"):
        o.integrate_state(rho_of(m, P_ATM, 1200.0, Y0), np.r_[Y0, 1200.0], -1e-7)


def test_trajectory_table_is_ignition_trajectories():
    """data/ (written by tools/make_trajectories.py from the oracle): every stored trajectory has
    tau > 0 and burns (T rises > 400 K by 2 tau), including the cool jisc shear-layer mixtures."""
    import synth
    doc = synth.load_trajectories()
    for tr in doc["trajectories"]:
        assert tr["tau"] > 0.0, tr.get("Z")
        f = np.asarray(tr["t_over_tau"])
        T = np.asarray(tr["T"])
        assert T[np.searchsorted(f, 2.0)] - tr["T0"] > 400.0, (tr["kind"], tr.get("Z"))

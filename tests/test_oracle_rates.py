"""Pins for the oracle's rates and Jacobian (SURVEY.md §8(c) "Rates: identity / trivial cases /
conservation", "K_c and thermo", "Jacobian")."""
import numpy as np

from oracle import Oracle
from tests.pins.matrix_rates import gross, matrix_rates

R = 8.314462618


def _random_states(m, n, seed):
    """cfg1d recipe: T ~ U[300,3000], p ~ logU[0.1,100] atm, Y ~ Dirichlet(0.5)
    with 20% of entries zeroed and renormalised."""
    rng = np.random.default_rng(seed)
    T = rng.uniform(300, 3000, n)
    p = 101325.0 * 10 ** rng.uniform(-1, 2, n)
    Y = rng.dirichlet(0.5 * np.ones(m.ns), n)
    Y[rng.random((n, m.ns)) < 0.2] = 0.0
    Y[Y.sum(1) == 0, -1] = 1.0
    Y /= Y.sum(1, keepdims=True)
    rho = p / (R * T * np.sum(Y / m.W, axis=1))
    return rho, T, Y


def test_loop_equals_matrix_form(oracle_h2):
    """Oracle per-reaction loop (pow/products) == independent numpy ln-space matrix form."""
    m = oracle_h2.m
    rho, T, Y = _random_states(m, 400, 11)
    w_mat, qf_mat, qr_mat = matrix_rates(m, rho, T, Y)
    G = gross(m, qf_mat, qr_mat)
    for i in range(len(rho)):
        w, qf, qr = oracle_h2.rates(rho[i], T[i], Y[i])
        assert np.all(np.abs(w - w_mat[i]) <= 1e-12 * G[i] + 1e-300), i
        assert np.allclose(qf, qf_mat[i], rtol=1e-12, atol=0)
        assert np.allclose(qr, qr_mat[i], rtol=1e-12, atol=0)


def test_a_to_b_trivial():
    """A->B, A=1e3, Ea=0, [A]=1 mol/m^3 -> Omega_A = -1000, Omega_B = +1000."""
    o = Oracle("toy_a_to_b")
    W = o.m.W[0]
    rho = 1.0 * W / 1.0          # Y_A = 1 -> [A] = rho/W = 1
    w, _, _ = o.rates(rho, 700.0, np.array([1.0, 0.0]))
    assert w[0] == -1000.0 and w[1] == 1000.0


def test_inert_composition_zero(oracle_h2):
    """only non-reacting species -> Omega = 0 exactly."""
    Y = np.zeros(9)
    Y[-1] = 1.0
    w, _, _ = oracle_h2.rates(1.0, 1500.0, Y)
    assert np.all(w == 0.0)


def test_mass_and_element_conservation(oracle_h2):
    """sum_k W_k Omega_k = 0 and sum_k a_ek Omega_k = 0 relative to gross sums."""
    m = oracle_h2.m
    rho, T, Y = _random_states(m, 300, 12)
    for i in range(len(rho)):
        w, qf, qr = oracle_h2.rates(rho[i], T[i], Y[i])
        G = gross(m, qf[None], qr[None])[0]
        assert abs(np.dot(m.W, w)) <= 1e-12 * np.dot(m.W, G) + 1e-300
        for e in range(m.comp.shape[1]):
            a = m.comp[:, e].astype(float)
            assert abs(np.dot(a, w)) <= 1e-12 * np.dot(a, G) + 1e-300


def test_jacobian_complex_step_vs_finite_difference(oracle_h2):
    """The complex-step Jacobian agrees with central differences of the RHS (to FD accuracy)."""
    m = oracle_h2.m
    rho, T, Y = _random_states(m, 8, 13)
    for i in range(len(rho)):
        y = np.r_[Y[i] + 1e-6, T[i]]              # keep away from the max(Y,0) kink
        J = oracle_h2.jac(rho[i], y)
        n = len(y)
        Jfd = np.zeros((n, n))
        for j in range(n):
            hstep = 1e-6 * max(abs(y[j]), 1e-3)
            yp, ym = y.copy(), y.copy()
            yp[j] += hstep
            ym[j] -= hstep
            Jfd[:, j] = (oracle_h2.rhs(rho[i], yp) - oracle_h2.rhs(rho[i], ym)) / (2 * hstep)
        scale = np.abs(J).max(axis=1, keepdims=True) + 1e-300
        assert np.max(np.abs(J - Jfd) / scale) < 1e-5


def test_rhs_sums(oracle_h2):
    """Eq. 5: sum_k dY_k/dt = sum_k W_k Omega_k / rho = 0 (mass conservation)."""
    m = oracle_h2.m
    rho, T, Y = _random_states(m, 100, 14)
    for i in range(len(rho)):
        f = oracle_h2.rhs(rho[i], np.r_[Y[i], T[i]])
        w, qf, qr = oracle_h2.rates(rho[i], T[i], Y[i])
        G = gross(m, qf[None], qr[None])[0]
        assert abs(f[:-1].sum()) <= 1e-12 * np.dot(m.W, G) / rho[i] + 1e-300

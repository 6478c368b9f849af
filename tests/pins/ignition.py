"""Ignition-delay and equilibrium helpers for the oracle pins (test code only).

tau_ign = time of max dT/dt (SURVEY reading 16), located on a sampled
grid and refined by a parabola through the three samples around the maximum.

equilibrium_uv: constant-(u, v) chemical equilibrium from thermo and element composition only
(element-potential form): at equilibrium mu_k/RT = sum_e lambda_e a_ek, i.e.
c_k = (p0/(R T)) exp(sum_e lambda_e a_ek - g_k(T)), subject to element conservation
sum_k a_ek c_k = b_e and energy conservation sum_k c_k eps_k(T) = rho e.  No kinetics, no K_c.
"""
import numpy as np

from oracle.ignition import ignition_delay, trajectory  # noqa: F401

from tests.pins.matrix_rates import nasa

R = 8.314462618
P0 = 101325.0


def fresh_Y(m, phi=1.0):
    """phi=1 H2-air, O2:N2 = 1:3.76 by moles (SURVEY reading 18)."""
    X = np.zeros(m.ns)
    X[m.species.index("H2")] = 2.0 * phi
    X[m.species.index("O2")] = 1.0
    X[m.species.index("N2")] = 3.76
    Y = X * m.W
    return Y / Y.sum()


def rho_of(m, p, T, Y):
    return p / (R * T * np.sum(Y / m.W))


def _element_potentials(m, T, b):
    """At fixed T, minimise the convex dual phi(lam) = sum_k c_k(lam) - b.lam whose stationarity
    condition is element conservation A^T c(lam) = b."""
    A = m.comp.astype(float)
    cpR, hRT, sR = nasa(m, np.array([T]))
    g = (hRT - sR)[0]
    pref = P0 / (R * T)
    lam = np.zeros(A.shape[1])
    lam = np.log(b / pref) - 0.0   # rough start
    for _ in range(200):
        z = np.minimum(A @ lam - g, 700.0)
        c = pref * np.exp(z)
        grad = A.T @ c - b
        H = A.T @ (c[:, None] * A)
        step = np.linalg.solve(H, grad)
        phi0 = c.sum() - b @ lam
        t = 1.0
        while t > 1e-12:
            ln = lam - t * step
            cn = pref * np.exp(np.minimum(A @ ln - g, 700.0))
            if cn.sum() - b @ ln <= phi0 - 1e-4 * t * grad @ step:
                break
            t *= 0.5
        lam = ln
        if np.max(np.abs(grad) / b) < 1e-15 or np.max(np.abs(t * step)) < 1e-15:
            break
    c = pref * np.exp(A @ lam - g)
    return c, hRT[0]


def equilibrium_uv(m, rho, e, Y0):
    """Return (T_eq, Y_eq, element residual) of the constant-(u, v) equilibrium state."""
    from scipy.optimize import brentq
    b = rho * (Y0 / m.W) @ m.comp                     # element moles per volume [ne]

    def energy_resid(T):
        c, hRT = _element_potentials(m, T, b)
        return c @ ((hRT - 1.0) * R * T) - rho * e

    T = brentq(energy_resid, 1000.0, 4500.0, xtol=1e-13, rtol=1e-15, maxiter=500)
    c, _ = _element_potentials(m, T, b)
    Y = c * m.W / rho
    return T, Y, np.max(np.abs(m.comp.T.astype(float) @ c - b) / b)

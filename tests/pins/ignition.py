"""Ignition-delay and equilibrium helpers for the oracle pins (test code only).

tau_ign = time of max dT/dt (SURVEY reading 16), located on a sampled
grid and refined by a parabola through the three samples around the maximum.

equilibrium_uv: constant-(u, v) chemical equilibrium from thermo and element composition only
(element-potential form): at equilibrium mu_k/RT = sum_e lambda_e a_ek, i.e.
c_k = (p0/(R T)) exp(sum_e lambda_e a_ek - g_k(T)), subject to element conservation
sum_k a_ek c_k = b_e and energy conservation sum_k c_k eps_k(T) = rho e.  No kinetics, no K_c.
"""
import numpy as np

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


def trajectory(o, rho, y0, times, rtol=1e-12, atolY=1e-24, atolT=1e-9):
    """States at the given increasing times (restarting the integrator at each output)."""
    out = [np.array(y0, dtype=float)]
    y = np.array(y0, dtype=float)
    t = 0.0
    for tn in times[1:]:
        y, _ = o.integrate_state(rho, y, tn - t, rtol, atolY, atolT)
        out.append(y.copy())
        t = tn
    return np.array(out)


def ignition_delay(o, rho, y0, t_end, n_coarse=200, n_fine=80, rtol=1e-10):
    """Two passes: locate max dT/dt on [0, t_end], then resample [0, 2 tau_1] and refine."""
    tau1 = _ignition_pass(o, rho, y0, t_end, n_coarse, n_fine, rtol)
    return _ignition_pass(o, rho, y0, 2.0 * tau1, n_coarse, n_fine, rtol)


def _ignition_pass(o, rho, y0, t_end, n_coarse, n_fine, rtol):
    ts = np.linspace(0.0, t_end, n_coarse + 1)
    ys = trajectory(o, rho, y0, ts, rtol=rtol)
    dT = np.array([o.rhs(rho, y)[-1] for y in ys])
    i = int(np.argmax(dT))
    i = min(max(i, 1), n_coarse - 1)
    # refine on [t_{i-1}, t_{i+1}]
    tf = np.linspace(ts[i - 1], ts[i + 1], n_fine + 1)
    yf = [ys[i - 1]]
    y = ys[i - 1].copy()
    for a, b in zip(tf[:-1], tf[1:]):
        y, _ = o.integrate_state(rho, y, b - a, rtol, 1e-24, 1e-9)
        yf.append(y.copy())
    dTf = np.array([o.rhs(rho, y)[-1] for y in yf])
    j = int(np.argmax(dTf))
    j = min(max(j, 1), n_fine - 1)
    x0, x1, x2 = tf[j - 1], tf[j], tf[j + 1]
    f0, f1, f2 = dTf[j - 1], dTf[j], dTf[j + 1]
    denom = f0 - 2 * f1 + f2
    if denom == 0:
        return x1
    return x1 + 0.5 * (x1 - x0) * (f0 - f2) / denom


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

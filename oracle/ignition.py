"""Ignition delay and trajectory sampling on the oracle (TEST INFRASTRUCTURE ONLY).

tau_ign = time of max dT/dt (SURVEY reading 16), located on a sampled grid
and refined by a parabola through the three samples around the maximum (two passes: locate on
[0, t_end], then resample [0, 2 tau_1]).  Trajectories restart the oracle's BDF at each output
time (exact outputs, no dense-output interpolation).
"""
import numpy as np


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



"""Ignition delay and trajectory sampling on the oracle (TEST INFRASTRUCTURE ONLY).

tau_ign = time of max dT/dt (SURVEY reading 16), located on a sampled grid
and refined by a parabola through the three samples around the maximum (two passes: locate on
[0, t_end], then resample [0, 2 tau_1]).  Trajectories restart the oracle's BDF at each output
time (exact outputs, no dense-output interpolation).

An ignition is only reported when the maximum of dT/dt is INTERIOR to the sampled window and the
temperature has risen by at least `min_rise` K by the end of it; otherwise the window is doubled
(up to `t_max`) and, if no ignition is found, `NoIgnition` is raised.  (Round 1 clamped a maximum
at t = 0 to the first interior sample and extrapolated a negative tau.)
"""
import numpy as np


class NoIgnition(RuntimeError):
    """The mixture does not ignite (no interior max of dT/dt with a temperature rise) in t_max."""


def trajectory(o, rho, y0, times, rtol=1e-12, atolY=1e-24, atolT=1e-9):
    """States at the given increasing times (restarting the integrator at each output)."""
    times = np.asarray(times, dtype=float)
    if np.any(np.diff(times) < 0) or times[0] != 0.0:
        raise ValueError("trajectory times must start at 0 and be non-decreasing")
    out = [np.array(y0, dtype=float)]
    y = np.array(y0, dtype=float)
    t = 0.0
    for tn in times[1:]:
        y, _ = o.integrate_state(rho, y, tn - t, rtol, atolY, atolT)
        out.append(y.copy())
        t = tn
    return np.array(out)


def ignition_delay(o, rho, y0, t_end, n_coarse=200, n_fine=80, rtol=1e-10, min_rise=50.0, t_max=1.0):
    """Two passes: locate an interior max dT/dt on [0, t_end] (doubling t_end up to t_max until one
    exists), then resample [0, 2 tau_1] and refine.  Raises NoIgnition when there is none."""
    while True:
        tau1 = _ignition_pass(o, rho, y0, t_end, n_coarse, n_fine, rtol, min_rise)
        if tau1 is not None:
            break
        t_end *= 2.0
        if t_end > t_max:
            raise NoIgnition(f"no ignition within {t_max} s (T0 = {y0[-1]:.1f} K)")
    tau = _ignition_pass(o, rho, y0, 2.0 * tau1, n_coarse, n_fine, rtol, min_rise)
    if tau is None or not (0.0 < tau < 2.0 * tau1):
        raise NoIgnition(f"refinement lost the ignition found at {tau1:.3e} s")
    return tau


def _ignition_pass(o, rho, y0, t_end, n_coarse, n_fine, rtol, min_rise):
    """tau on [0, t_end], or None if the maximum of dT/dt is not interior or T did not rise."""
    ts = np.linspace(0.0, t_end, n_coarse + 1)
    ys = trajectory(o, rho, y0, ts, rtol=rtol)
    dT = np.array([o.rhs(rho, y)[-1] for y in ys])
    i = int(np.argmax(dT))
    if i == 0 or i == n_coarse or ys[-1, -1] - ys[0, -1] < min_rise:
        return None
    # refine on [t_{i-1}, t_{i+1}]
    tf = np.linspace(ts[i - 1], ts[i + 1], n_fine + 1)
    yf = [ys[i - 1]]
    y = ys[i - 1].copy()
    for a, b in zip(tf[:-1], tf[1:]):
        y, _ = o.integrate_state(rho, y, b - a, rtol, 1e-24, 1e-9)
        yf.append(y.copy())
    dTf = np.array([o.rhs(rho, y)[-1] for y in yf])
    j = int(np.argmax(dTf))
    if j == 0 or j == n_fine:
        return None
    x0, x1, x2 = tf[j - 1], tf[j], tf[j + 1]
    f0, f1, f2 = dTf[j - 1], dTf[j], dTf[j + 1]
    denom = f0 - 2 * f1 + f2
    if denom >= 0:          # not a strict local maximum of the sampled parabola
        return x1
    return x1 + 0.5 * (x1 - x0) * (f0 - f2) / denom

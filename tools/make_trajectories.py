"""Write data/trajectories_h2air_li2004.json: the reactor-trajectory states the synthetic inputs
sample from (SURVEY.md §8(d) "Reactor-trajectory states are 0-D oracle states sampled along a
constant-volume run from the stated initial condition").

Calls only oracle/ (and synth's composition helpers, which hold no method arithmetic).  The
stored numbers are INPUTS for both sides, never expected values.

    python tools/make_trajectories.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from oracle import Oracle  # noqa: E402
from oracle.ignition import ignition_delay, trajectory  # noqa: E402

TOL = dict(rtol=1e-12, atolY=1e-24, atolT=1e-9)
FRACS = np.linspace(0.0, 3.0, 241)          # t / tau samples


def _traj(o, rho, Y0, T0, t_end_guess, **meta):
    y0 = np.r_[Y0, T0]
    tau = ignition_delay(o, rho, y0, t_end_guess)      # raises NoIgnition if there is none
    ys = trajectory(o, rho, y0, FRACS * tau, **TOL)
    # the stored states must be an ignition trajectory: tau > 0, T rises through the window
    assert tau > 0.0, (meta, tau)
    assert ys[-1, -1] - T0 > 400.0, (meta, T0, ys[-1, -1])
    assert ys[FRACS.searchsorted(2.0), -1] - T0 > 400.0, (meta, "not burnt by 2 tau")
    return dict(meta, rho=float(rho), tau=float(tau), T0=float(T0), t_over_tau=FRACS.tolist(),
                T=ys[:, -1].tolist(), Y=ys[:, :-1].tolist())


def enthalpy(o, T, Y):
    """h = u + R T / Wbar (J/kg)."""
    return o.energy(T, Y) + synth.R_GAS * T * np.sum(Y / o.m.W)


def T_from_h(o, h, Y, T):
    for _ in range(100):
        cp = o.cv(T, Y) + synth.R_GAS * np.sum(Y / o.m.W)
        dT = (enthalpy(o, T, Y) - h) / cp
        T -= dT
        if abs(dT) < 1e-12 * T:
            return T
    raise RuntimeError("enthalpy Newton failed")


def main():
    o = Oracle("h2air_li2004")
    m = o.m
    Yf = synth.fresh_Y(m.species, m.W)
    out = dict(mechanism="h2air_li2004", species=m.species, generated_by="tools/make_trajectories.py",
               oracle_tolerances=TOL, trajectories=[])
    # fresh phi=1, 1 atm (cfg1b, cfg2)
    for T0 in (1000.0, 1100.0, 1200.0, 1300.0, 1400.0, 1500.0):
        rho = synth.rho_ideal(synth.P_ATM, T0, Yf, m.W)[0]
        out["trajectories"].append(_traj(o, rho, Yf, T0, 3e-3, kind="fresh", p0=synth.P_ATM))
        print("fresh", T0, out["trajectories"][-1]["tau"])
    # von Neumann state of a CJ H2-air detonation (approximate textbook values)
    T_vn, p_vn = 1530.0, 28.0 * synth.P_ATM
    rho = synth.rho_ideal(p_vn, T_vn, Yf, m.W)[0]
    out["trajectories"].append(_traj(o, rho, Yf, T_vn, 1e-4, kind="vN", p0=p_vn))
    print("vN", out["trajectories"][-1]["tau"])
    # jet in crossflow mixing line (cfg5): pure H2 at 250 K into air at 1200 K, (Y, h) linear in Z
    Yj = np.zeros(m.ns); Yj[m.species.index("H2")] = 1.0
    Ya = synth.air_Y(m.species, m.W)
    Tj, Ta = 250.0, 1200.0
    hj, ha = enthalpy(o, Tj, Yj), enthalpy(o, Ta, Ya)
    Zs = np.linspace(0.0, 1.0, 2001)
    Tm, rm = [], []
    T = Ta
    for Z in Zs:
        Y = Z * Yj + (1 - Z) * Ya
        T = T_from_h(o, Z * hj + (1 - Z) * ha, Y, T)
        Tm.append(T)
        rm.append(synth.rho_ideal(synth.P_ATM, T, Y, m.W)[0])
    out["jisc_mixing"] = dict(Z=Zs.tolist(), T=Tm, rho=rm, Y_jet=Yj.tolist(), Y_air=Ya.tolist(), T_jet=Tj, T_air=Ta)
    # shear-layer reaction-zone trajectories of the mixed gas, Z in |Z - Z_st| < 0.01
    Z_st = 0.0285
    for Z in np.linspace(Z_st - 0.01, Z_st + 0.01, 9):
        Y = Z * Yj + (1 - Z) * Ya
        T0 = T_from_h(o, Z * hj + (1 - Z) * ha, Y, Ta)
        rho = synth.rho_ideal(synth.P_ATM, T0, Y, m.W)[0]
        out["trajectories"].append(_traj(o, rho, Y, T0, 3e-3, kind="jisc_shear", Z=float(Z), p0=synth.P_ATM))
        print("shear", Z, T0, out["trajectories"][-1]["tau"])
    path = os.path.join(ROOT, "data", "trajectories_h2air_li2004.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=None, separators=(",", ":"))
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()

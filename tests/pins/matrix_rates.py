"""Independent numpy matrix-form rate evaluation (SURVEY.md §8(a) A4 block), used as a pin
for the oracle's per-reaction loop (SURVEY.md §8(c) "Rates: identity"
"standalone rate-evaluation oracle").

Matrix form (BASELINE.json north_star, "ln k from T, forward/reverse rates as exp of
stoichiometry-matrix products with ln c, net production via the (nu''-nu') matrix"):

  ln kf = ln A + b ln T - Ea/(R T)
  ln c  = log(rho max(Y,0)/W)            (log 0 = -inf; only nonzero nu entries are summed)
  ln Kc = -nu^T g + (sum nu) ln(p0/(R T)),  g = h/RT - s/R
  ln qf = ln kf + nu'^T ln c ;  ln qr = ln kf - ln Kc + nu''^T ln c
  q     = (exp ln qf - exp ln qr) * ([M] or falloff factor)
  Omega = (nu'' - nu') q

Vectorised over cells with masked products (no 0 * -inf).  Thermo is evaluated here from the
NASA-7 definition independently of the oracle's C code.
"""
import numpy as np

R = 8.314462618
P0 = 101325.0


def nasa(m, T):
    """cp/R, h/RT, s/R arrays [ncell, ns] for temperatures T [ncell]."""
    T = np.asarray(T, dtype=np.float64)[:, None]
    lo = T < m.T_range[None, :, 1]
    a = np.where(lo[..., None], m.nasa_lo[None], m.nasa_hi[None])     # [n, ns, 7]
    a1, a2, a3, a4, a5, a6, a7 = (a[..., i] for i in range(7))
    cpR = a1 + T * (a2 + T * (a3 + T * (a4 + T * a5)))
    hRT = a1 + T * (a2 / 2 + T * (a3 / 3 + T * (a4 / 4 + T * a5 / 5))) + a6 / T
    sR = a1 * np.log(T) + T * (a2 + T * (a3 / 2 + T * (a4 / 3 + T * a5 / 4))) + a7
    return cpR, hRT, sR


def masked_matvec(lnc, nu):
    """sum_k nu[r,k] lnc[:,k] over nonzero nu only -> [n, nr]."""
    out = np.zeros((lnc.shape[0], nu.shape[0]))
    for r in range(nu.shape[0]):
        for k in np.nonzero(nu[r])[0]:
            out[:, r] += nu[r, k] * lnc[:, k]
    return out


def matrix_rates(m, rho, T, Y):
    """Return (wdot [n, ns], qf [n, nr], qr [n, nr]) with [M]/falloff factors folded into q."""
    rho = np.asarray(rho, dtype=np.float64)
    T = np.asarray(T, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    lnT = np.log(T)[:, None]
    invT = 1.0 / T[:, None]
    c = rho[:, None] * np.maximum(Y, 0.0) / m.W[None, :]
    with np.errstate(divide="ignore"):
        lnc = np.log(c)
    lnkf = np.log(m.A)[None] + m.b[None] * lnT - (m.Ea[None] / R) * invT
    M = c @ m.eff.T                                                # [n, nr]
    fo = (m.kind == 2) | (m.kind == 3)
    if np.any(fo):
        with np.errstate(divide="ignore"):
            lnk0 = np.log(np.where(m.A0 > 0, m.A0, 1.0))[None] + m.b0[None] * lnT - (m.Ea0[None] / R) * invT
        Pr = np.exp(lnk0 - lnkf) * M
        F = np.ones_like(Pr)
        tr = m.kind == 3
        if np.any(tr):
            al, T3, T1, T2 = (m.troe[:, i][None] for i in range(4))
            Tc = T[:, None]
            with np.errstate(over="ignore"):
                Fc = (1 - al) * np.exp(-Tc / np.where(T3 != 0, T3, 1.0)) + al * np.exp(-Tc / np.where(T1 != 0, T1, 1.0))
                Fc = Fc + np.where(T2 > 0, np.exp(-np.where(T2 > 0, T2, 0.0) / Tc), 0.0)
            with np.errstate(divide="ignore", invalid="ignore"):
                lFc = np.log10(Fc)
                lPr = np.log10(Pr)
                C = -0.4 - 0.67 * lFc
                N = 0.75 - 1.27 * lFc
                f1 = (lPr + C) / (N - 0.14 * (lPr + C))
                Ftr = 10.0 ** (lFc / (1 + f1 * f1))
            F = np.where(tr[None], Ftr, F)
        lnfac = np.log(Pr / (1 + Pr) * F)
        lnkf = np.where(fo[None], lnkf + lnfac, lnkf)
    cpR, hRT, sR = nasa(m, T)
    g = hRT - sR
    nu = (m.nu_r - m.nu_f).astype(np.float64)
    dnu = nu.sum(axis=1)
    lnKc = -(g @ nu.T) + dnu[None] * np.log(P0 / (R * T))[:, None]
    lnqf = lnkf + masked_matvec(lnc, m.nu_f.astype(np.float64))
    lnqr = lnkf - lnKc + masked_matvec(lnc, m.nu_r.astype(np.float64))
    qf = np.exp(lnqf)
    qr = np.where(m.reversible[None] == 1, np.exp(lnqr), 0.0)
    tb = (m.kind == 1)[None]
    qf = np.where(tb, qf * M, qf)
    qr = np.where(tb, qr * M, qr)
    wdot = (qf - qr) @ nu
    return wdot, qf, qr


def gross(m, qf, qr):
    nu = np.abs(m.nu_r - m.nu_f).astype(np.float64)
    return (np.abs(qf) + np.abs(qr)) @ nu

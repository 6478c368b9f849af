"""The CPU oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import, call, link or execute anything under ``oracle/``.  The
product path (``paper_2510_23993_b200``) never imports it and shares no code with it: no kernels,
headers, helpers, tables, constant generators, pre- or post-processing.  Only the mechanism data
files under ``mech/`` and the seeded input generators (``synth/``, no method arithmetic) are
common to both.

What the oracle computes (§2.1):
  * thermo (NASA-7), T from (e, Y) by Newton at constant (e, rho)            — chem_oracle.c
  * per-reaction-loop rates with pow/products (not ln-space), third-body,
    Lindemann/Troe falloff, K_c from NASA Gibbs                              — oracle_rhs.inc
  * RHS of Eq. 5 and the corrected Eq. 6                                      — oracle_rhs.inc
  * dense variable-order BDF, complex-step Jacobian, dense LU                 — chem_oracle.c
  * the Alg. 2/3 gate (T < T_min or solid -> untouched), T_out = Newton(e, Y_out)

Pins (what fixes the oracle other than itself) live in tests/test_oracle_*.py.

Parity unpinned: absolute kinetic parameters of the bundled Li et al. 2004 mechanism (no
Cantera offline, PAPER.md prints no rate values, only R^2 at P:458); see DESIGN.md.
"""
from __future__ import annotations

import ctypes
import os
import pathlib
import subprocess

import numpy as np

from . import mechanism as _mech

_HERE = pathlib.Path(__file__).resolve().parent
_SO = _HERE / "liboracle.so"
_SRC = [_HERE / "chem_oracle.c", _HERE / "oracle_rhs.inc"]

R_GAS = _mech.R_GAS
P_REF = _mech.P_REF
load_mechanism = _mech.load


def build(force: bool = False) -> pathlib.Path:
    """Compile liboracle.so with gcc -O3 -march=native -fopenmp."""
    if not force and _SO.exists() and all(_SO.stat().st_mtime >= s.stat().st_mtime for s in _SRC):
        return _SO
    tmp = _SO.with_suffix(f".{os.getpid()}.tmp")
    # -march=native is deliberately avoided: the .so travels to the GPU box whose host CPU may
    # differ from this one.  -O3 with the x86-64-v2 baseline is portable.
    cmd = ["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-o", str(tmp), str(_SRC[0]), "-lm"]
    subprocess.run(cmd, check=True, cwd=_HERE)
    os.replace(tmp, _SO)
    return _SO


class _OMech(ctypes.Structure):
    _fields_ = [("ns", ctypes.c_int32), ("nr", ctypes.c_int32)] + [
        (n, ctypes.c_void_p) for n in
        ("W", "Trange", "lo", "hi", "nu_f", "nu_r", "A", "b", "Ea", "kind", "rev", "eff",
         "A0", "b0", "Ea0", "troe")] + [("R", ctypes.c_double), ("p0", ctypes.c_double)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(str(_SO))
        P = ctypes.c_void_p
        D = ctypes.c_double
        lib.or_thermo.argtypes = [P, D, P, P, P]
        lib.or_rates.argtypes = [P, D, D, P, P, P, P]
        lib.or_rhs.argtypes = [P, D, P, P]
        lib.or_jac.argtypes = [P, D, P, P]
        lib.or_energy.argtypes = [P, D, P]
        lib.or_energy.restype = D
        lib.or_cv.argtypes = [P, D, P]
        lib.or_cv.restype = D
        lib.or_newton_T.argtypes = [P, D, P, D, P]
        lib.or_newton_T.restype = ctypes.c_int
        lib.or_integrate_state.argtypes = [P, D, P, D, D, D, D, P]
        lib.or_integrate_state.restype = ctypes.c_int
        lib.or_integrate_cells.argtypes = [P, ctypes.c_int64, P, P, P, P, P, D, D, D, D, D,
                                           ctypes.c_int, P, P, P]
        lib.or_max_threads.restype = ctypes.c_int
        lib.or_explicit_cells.argtypes = [P, ctypes.c_int64, P, P, P, P, P, D, D, D, ctypes.c_int64, ctypes.c_int,
                                          P, P]
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


class Oracle:
    """Slow, obviously-correct CPU reference for one mechanism."""

    def __init__(self, mech="h2air_li2004"):
        self.m = mech if isinstance(mech, _mech.OracleMechanism) else _mech.load(mech)
        m = self.m
        self._keep = [np.ascontiguousarray(x) for x in (
            m.W, m.T_range, m.nasa_lo, m.nasa_hi, m.nu_f.astype(np.int64), m.nu_r.astype(np.int64),
            m.A, m.b, m.Ea, m.kind.astype(np.int64), m.reversible.astype(np.int64), m.eff,
            m.A0, m.b0, m.Ea0, m.troe)]
        self._s = _OMech(m.ns, m.nr, *[_ptr(x) for x in self._keep], R_GAS, P_REF)
        self._sp = ctypes.cast(ctypes.pointer(self._s), ctypes.c_void_p)
        self.lib = _load()
        self.ns = m.ns
        self.nr = m.nr

    # ---- point functions -------------------------------------------------------------
    def thermo(self, T):
        cp, h, s = (np.zeros(self.ns) for _ in range(3))
        self.lib.or_thermo(self._sp, float(T), _ptr(cp), _ptr(h), _ptr(s))
        return cp, h, s

    def rates(self, rho, T, Y):
        """Return (wdot [ns] mol/m^3/s, qf [nr], qr [nr])."""
        Y = np.ascontiguousarray(Y, dtype=np.float64)
        w, qf, qr = np.zeros(self.ns), np.zeros(self.nr), np.zeros(self.nr)
        self.lib.or_rates(self._sp, float(rho), float(T), _ptr(Y), _ptr(w), _ptr(qf), _ptr(qr))
        return w, qf, qr

    def gross(self, rho, T, Y):
        """Gross species rate G_k = sum_r |nu_kr| (|qf_r| + |qr_r|) (SURVEY reading 13)."""
        _, qf, qr = self.rates(rho, T, Y)
        nu = np.abs(self.m.nu_r - self.m.nu_f).astype(np.float64)
        return nu.T @ (np.abs(qf) + np.abs(qr))

    def rhs(self, rho, y):
        y = np.ascontiguousarray(y, dtype=np.float64)
        f = np.zeros(self.ns + 1)
        self.lib.or_rhs(self._sp, float(rho), _ptr(y), _ptr(f))
        return f

    def jac(self, rho, y):
        y = np.ascontiguousarray(y, dtype=np.float64)
        n = self.ns + 1
        J = np.zeros((n, n))
        self.lib.or_jac(self._sp, float(rho), _ptr(y), _ptr(J))
        return J

    def energy(self, T, Y):
        Y = np.ascontiguousarray(Y, dtype=np.float64)
        return self.lib.or_energy(self._sp, float(T), _ptr(Y))

    def cv(self, T, Y):
        Y = np.ascontiguousarray(Y, dtype=np.float64)
        return self.lib.or_cv(self._sp, float(T), _ptr(Y))

    def newton_T(self, e, Y, T_guess):
        Y = np.ascontiguousarray(Y, dtype=np.float64)
        out = ctypes.c_double(0.0)
        it = self.lib.or_newton_T(self._sp, float(e), _ptr(Y), float(T_guess), ctypes.byref(out))
        return out.value, it

    def energies(self, T, Y):
        """e_i = u(T_i, Y_i) for cell-major Y [n, ns]."""
        return np.array([self.energy(t, y) for t, y in zip(np.asarray(T), np.asarray(Y))])

    # ---- integration -----------------------------------------------------------------
    def integrate_state(self, rho, y0, tf, rtol=1e-12, atolY=1e-24, atolT=1e-9):
        """One reactor state y=(Y,T) over [0, tf]; returns (y, stats[steps, rej, nfev, njev, nlu])."""
        y = np.array(y0, dtype=np.float64)
        st = np.zeros(5, dtype=np.int64)
        rc = self.lib.or_integrate_state(self._sp, float(rho), _ptr(y), float(tf), rtol, atolY, atolT, _ptr(st))
        if rc != 0:
            raise RuntimeError(f"oracle BDF failed rc={rc}")
        return y, st

    def integrate_cells(self, rho, e, T, Y, dt, rtol=1e-12, atolY=1e-24, atolT=1e-9, T_min=500.0,
                        solid=None, nthreads=None):
        """The gated cell loop.  Y is cell-major [n, ns].

        Returns dict(T, Y, status, nsteps, T_int)."""
        n = len(rho)
        rho = np.ascontiguousarray(rho, dtype=np.float64)
        e = np.ascontiguousarray(e, dtype=np.float64)
        T = np.array(T, dtype=np.float64)
        Y = np.array(Y, dtype=np.float64, order="C").reshape(n, self.ns)
        sol = None if solid is None else np.ascontiguousarray(solid, dtype=np.uint8)
        nst = np.zeros(n, dtype=np.int64)
        status = np.zeros(n, dtype=np.int32)
        T_int = np.zeros(n)
        nth = nthreads or self.lib.or_max_threads()
        self.lib.or_integrate_cells(self._sp, n, _ptr(rho), _ptr(e), _ptr(T), _ptr(Y), _ptr(sol), float(dt),
                                    rtol, atolY, atolT, T_min, int(nth), _ptr(nst), _ptr(status), _ptr(T_int))
        return dict(T=T, Y=Y, status=status, nsteps=nst, T_int=T_int, threads=nth)

    def explicit_cells(self, rho, e, T, Y, dt, eps=0.01, T_min=500.0, kmax=100000, solid=None, nthreads=None):
        """The paper's explicit scheme over cell-major Y [n, ns]."""
        n = len(rho)
        rho = np.ascontiguousarray(rho, dtype=np.float64)
        e = np.ascontiguousarray(e, dtype=np.float64)
        T = np.array(T, dtype=np.float64)
        Y = np.array(Y, dtype=np.float64, order="C").reshape(n, self.ns)
        sol = None if solid is None else np.ascontiguousarray(solid, dtype=np.uint8)
        nst = np.zeros(n, dtype=np.int64)
        status = np.zeros(n, dtype=np.int32)
        nth = nthreads or self.lib.or_max_threads()
        self.lib.or_explicit_cells(self._sp, n, _ptr(rho), _ptr(e), _ptr(T), _ptr(Y), _ptr(sol), float(dt),
                                   float(eps), float(T_min), int(kmax), int(nth), _ptr(nst), _ptr(status))
        return dict(T=T, Y=Y, status=status, nsteps=nst)

    def max_threads(self):
        return self.lib.or_max_threads()

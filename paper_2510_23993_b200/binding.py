"""ctypes binding of libchem.so (include/chem.h) — argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C ABI; this module converts
torch tensors to device pointers, picks the current CUDA stream, owns the workspace tensor and
translates return codes into exceptions.  There is no fallback: if libchem.so is missing or a
tensor is not on a CUDA device the calls raise.
"""
from __future__ import annotations

import ctypes
import pathlib

import numpy as np

from . import mechanism as _mech

LIB_PATH = pathlib.Path(__file__).resolve().parent / "libchem.so"

CHEM_METHOD_RODAS4 = 0
CHEM_METHOD_RODAS3 = 1
CHEM_METHOD_EXPLICIT = 2

# per-cell outcome codes of chem_cell_status
CHEM_CELL_UNTOUCHED, CHEM_CELL_DONE, CHEM_CELL_UNFINISHED, CHEM_CELL_FAILED = 0, 1, 2, -1

_ERRORS = {-1: "CHEM_EINVAL", -2: "CHEM_EMECH", -3: "CHEM_ENOSTRUCT", -4: "CHEM_ECUDA", -5: "CHEM_ENOWS"}


class ChemError(RuntimeError):
    def __init__(self, code, lib=None):
        msg = _ERRORS.get(code, str(code))
        if lib is not None:
            msg += ": " + lib.chem_strerror(code).decode()
        super().__init__(msg)
        self.code = code


class ChemMechDesc(ctypes.Structure):
    _fields_ = [("ns", ctypes.c_int32), ("nr", ctypes.c_int32), ("ne", ctypes.c_int32)] + [
        (n, ctypes.c_void_p) for n in ("W", "nasa_lo", "nasa_hi", "T_range", "elem", "nu_f", "nu_r", "A", "b", "Ea",
                                       "type", "reversible", "eff", "A0", "b0", "Ea0", "troe")] + [
        ("R", ctypes.c_double), ("p_ref", ctypes.c_double)]


class ChemOpts(ctypes.Structure):
    _fields_ = [("T_min", ctypes.c_double), ("kmax_bulk", ctypes.c_int32), ("n_active_star", ctypes.c_int64),
                ("kmax_sparse", ctypes.c_int32), ("atol_T", ctypes.c_double), ("method", ctypes.c_int32),
                ("compact_bulk", ctypes.c_int32), ("eps_change", ctypes.c_double), ("h0_factor", ctypes.c_double),
                ("lockstep", ctypes.c_int32), ("kmax_first", ctypes.c_int32), ("schedule_lpt", ctypes.c_int32)]


class ChemBox(ctypes.Structure):
    _fields_ = [("rho", ctypes.c_void_p), ("e", ctypes.c_void_p), ("T", ctypes.c_void_p), ("Y", ctypes.c_void_p),
                ("solid", ctypes.c_void_p), ("ncells", ctypes.c_int64), ("ld", ctypes.c_int64),
                ("dt", ctypes.c_double)]


class ChemStats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "cells", "active0", "bulk_iters", "sparse_cells", "steps_attempted", "steps_accepted", "steps_frozen", "rhs_evals",
        "jac_evals", "lu_count", "n_unfinished", "n_newton_fail", "n_nonfinite", "n_T_range")] + [
        (n, ctypes.c_double) for n in ("t_gate_ms", "t_bulk_ms", "t_compact_ms", "t_sparse_ms",
                                       "max_energy_drift")] + [("active_per_iter", ctypes.c_int64 * 16)] + [
        (n, ctypes.c_int64) for n in ("warp_substeps", "bulk_substeps", "lockstep", "lpt")] + [
        ("hint_accuracy", ctypes.c_double), ("kernel_launches", ctypes.c_int64)]

    def to_dict(self):
        d = {n: getattr(self, n) for n, _ in self._fields_ if n != "active_per_iter"}
        d["active_per_iter"] = list(self.active_per_iter)[: max(0, min(16, self.bulk_iters))]
        return d


# every symbol include/chem.h declares (checked by tests/test_cabi.py on CPU)
EXPORTED = ("chem_default_opts", "chem_init", "chem_finalize", "chem_strerror", "chem_structure_name",
            "chem_set_opts", "chem_workspace_bytes", "chem_rates", "chem_integrate", "chem_integrate_boxes",
            "chem_temperature", "chem_energy", "chem_jacobian", "chem_rhs", "chem_set_trace", "chem_internal_energy", "chem_cell_status", "chem_box_active")

_lib = None


def load_library():
    """Load libchem.so; raise if it is missing (no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2510_23993_b200.build` "
                           "(there is no fallback path)")
    lib = ctypes.CDLL(str(LIB_PATH))
    P, I64, D, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int32
    lib.chem_default_opts.argtypes = [P]
    lib.chem_default_opts.restype = None
    lib.chem_init.argtypes = [P, P, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
    lib.chem_finalize.argtypes = [P]
    lib.chem_finalize.restype = None
    lib.chem_strerror.argtypes = [ctypes.c_int]
    lib.chem_strerror.restype = ctypes.c_char_p
    lib.chem_structure_name.argtypes = [P]
    lib.chem_structure_name.restype = ctypes.c_char_p
    lib.chem_set_opts.argtypes = [P, P]
    lib.chem_workspace_bytes.argtypes = [P, I64, I32]
    lib.chem_workspace_bytes.restype = ctypes.c_size_t
    lib.chem_rates.argtypes = [P, I64, I64, P, P, P, P, P]
    lib.chem_rhs.argtypes = [P, I64, I64, P, P, P, P, P]
    lib.chem_jacobian.argtypes = [P, I64, I64, P, P, P, P, P]
    lib.chem_temperature.argtypes = [P, I64, I64, P, P, P, P]
    lib.chem_energy.argtypes = [P, I64, I64, P, P, P, P]
    lib.chem_integrate.argtypes = [P, I64, I64, P, P, P, P, P, D, D, D, P, ctypes.c_size_t, P, P]
    lib.chem_integrate_boxes.argtypes = [P, I32, P, D, D, P, ctypes.c_size_t, P, P, P]
    lib.chem_set_trace.argtypes = [P, P, I32]
    lib.chem_internal_energy.argtypes = [P, I64, I64, P, P, P]
    lib.chem_cell_status.argtypes = [P, P, ctypes.c_size_t, I64, I64, P, P, P]
    lib.chem_box_active.argtypes = [P, I32, P, P, P, ctypes.c_size_t, P]
    for f in ("chem_box_active", "chem_cell_status", "chem_init", "chem_set_opts", "chem_set_trace", "chem_internal_energy", "chem_rates", "chem_rhs", "chem_jacobian", "chem_temperature",
              "chem_energy", "chem_integrate", "chem_integrate_boxes"):
        getattr(lib, f).restype = ctypes.c_int
    _lib = lib
    return lib


def mech_desc(mt: _mech.MechTables):
    """Build a chem_mech_desc over numpy arrays; returns (desc, keepalive)."""
    arrs = dict(
        W=np.ascontiguousarray(mt.W, np.float64), nasa_lo=np.ascontiguousarray(mt.nasa_lo, np.float64),
        nasa_hi=np.ascontiguousarray(mt.nasa_hi, np.float64), T_range=np.ascontiguousarray(mt.T_range, np.float64),
        elem=np.ascontiguousarray(mt.elem, np.int32), nu_f=np.ascontiguousarray(mt.nu_f, np.float64),
        nu_r=np.ascontiguousarray(mt.nu_r, np.float64), A=np.ascontiguousarray(mt.A, np.float64),
        b=np.ascontiguousarray(mt.b, np.float64), Ea=np.ascontiguousarray(mt.Ea, np.float64),
        type=np.ascontiguousarray(mt.type, np.int32), reversible=np.ascontiguousarray(mt.reversible, np.int32),
        eff=np.ascontiguousarray(mt.eff, np.float64), A0=np.ascontiguousarray(mt.A0, np.float64),
        b0=np.ascontiguousarray(mt.b0, np.float64), Ea0=np.ascontiguousarray(mt.Ea0, np.float64),
        troe=np.ascontiguousarray(mt.troe, np.float64))
    d = ChemMechDesc()
    d.ns, d.nr, d.ne = mt.ns, mt.nr, mt.ne
    for k, a in arrs.items():
        setattr(d, k, a.ctypes.data)
    d.R = _mech.R_UNIVERSAL
    d.p_ref = _mech.P_STANDARD
    return d, arrs


def default_opts(lib=None) -> ChemOpts:
    lib = lib or load_library()
    o = ChemOpts()
    lib.chem_default_opts(ctypes.byref(o))
    return o

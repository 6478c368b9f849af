"""NEXT-3 on the CUDA path: the 14-species GRI-Mech 3.0 H/O/N/Ar mechanism (mech/gri30_hon.yaml)
through the same compiled kernels, against the oracle: rates (1e-10 gross-normalised, SURVEY reading
13), the analytic Jacobian (complex-step oracle, 1e-8), and integration over one dt at the parity
tolerance (T, Y_k > 1e-12 within 1e-6) on radical-rich H2-air states carrying NOx traces."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import Oracle  # noqa: E402
from paper_2510_23993_b200 import Chem  # noqa: E402
from tests.test_next3_mechanism import _states  # noqa: E402

DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module")
def ora():
    return Oracle("gri30_hon")


@pytest.fixture(scope="module")
def chem():
    return Chem("gri30_hon", device=0, atol_T=1e-6)


def dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device=DEV)


def test_structure(chem):
    assert chem.structure == "gri30_hon" and chem.ns == 14


def test_rates_and_jacobian_parity(chem, ora):
    m = ora.m
    rho, T, Y = _states(m, 1500, 21)                 # several tiles + a ragged tail
    w = chem.rates(dev(rho), dev(T), dev(Y.T)).cpu().numpy()
    for i in range(len(T)):
        wo, qf, qr = ora.rates(rho[i], T[i], Y[i])
        G = np.abs(m.nu_r - m.nu_f).T.astype(float) @ (np.abs(qf) + np.abs(qr))
        d = np.abs(w[:, i] - wo)
        assert np.all(d <= 1e-10 * G + 1e-300), i
        big = np.abs(wo) >= 1e-3 * G
        assert np.all(d[big] <= 1e-10 * np.abs(wo[big])), i
    Yp = (Y + 1e-8) / (Y + 1e-8).sum(1, keepdims=True)
    J = chem.jacobian(dev(rho[:128]), dev(T[:128]), dev(Yp[:128].T)).cpu().numpy()
    for i in range(128):
        Jo = ora.jac(rho[i], np.r_[Yp[i], T[i]])
        scale = np.abs(Jo).max(axis=1) + 1e-300
        assert (np.abs(J[:, :, i] - Jo).max(axis=1) / scale).max() < 1e-8, i


def _nox_states(m, n):
    """cfg1b-like radical-rich H2-air trajectory states (mapped by species name) with seeded NO, NO2,
    N2O, N traces (mole fraction 1e-6 .. 1e-3) and 1 % Ar by mole replacing N2."""
    doc = synth.load_trajectories()
    d = synth.cfg1b(doc, n=n)
    src = doc["species"]
    Y = np.zeros((n, m.ns))
    for j, s in enumerate(src):
        Y[:, m.species.index(s)] = d["Y"][:, j]
    rng = np.random.default_rng(31)
    for s, lo, hi in (("NO", 1e-5, 1e-3), ("NO2", 1e-7, 1e-5), ("N2O", 1e-7, 1e-5), ("N", 1e-9, 1e-7)):
        Y[:, m.species.index(s)] = 10 ** rng.uniform(np.log10(lo), np.log10(hi), n)
    iar, in2 = m.species.index("AR"), m.species.index("N2")
    Y[:, iar] = 0.013 * Y[:, in2]
    Y[:, in2] -= Y[:, iar]
    Y /= Y.sum(1, keepdims=True)
    return d["rho"], d["T"], Y, d["dt"]                 # the trajectory density (any rho > 0 is a state)


def test_integrate_parity(chem, ora):
    m = ora.m
    rho, T0, Y, dt = _nox_states(m, 512)
    e = np.array([ora.energy(t, y) for t, y in zip(T0, Y)])
    out = ora.integrate_cells(rho, e, T0, Y, dt, rtol=1e-12, atolY=1e-24, atolT=1e-9)
    assert np.all(out["status"] == 0)
    Td, Yd = dev(T0), dev(Y.T)
    st = chem.integrate(dev(rho), dev(e), Td, Yd, dt, rtol=1e-9, atol=1e-20)
    assert st["n_unfinished"] == 0 and st["n_nonfinite"] == 0
    Tg, Yg = Td.cpu().numpy(), Yd.cpu().numpy().T
    mask = out["Y"] > 1e-12
    assert np.max(np.abs(Tg / out["T"] - 1)) < 1e-6
    assert np.max(np.abs(Yg[mask] / out["Y"][mask] - 1)) < 1e-6
    # the inert Ar is untouched bitwise; N-species moved
    assert np.array_equal(Yg[:, m.species.index("AR")], Y[:, m.species.index("AR")])

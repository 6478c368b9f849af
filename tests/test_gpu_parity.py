"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element on the
same seeded inputs (BASELINE.json north_star tolerances; SURVEY.md §8(c) readings 13-14):

  * rates:      |Omega_gpu - Omega_ora| <= 1e-10 G_k (+1e-300), G_k the gross species rate,
                and plain relative 1e-10 wherever |Omega_k| >= 1e-3 G_k;
  * integration: T and Y_k (oracle Y_k > 1e-12) relative 1e-6 after one dt, GPU at the parity
                tolerance rtol = 1e-9, atol_Y = 1e-20, atol_T = 1e-6 K; oracle at rtol 1e-12,
                atol_Y 1e-24, atol_T 1e-9 K.
"""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import Oracle  # noqa: E402
from paper_2510_23993_b200 import Chem  # noqa: E402

DEV = torch.device("cuda", 0)
RTOL_RATES = 1e-10
RTOL_STATE = 1e-6
GPU_TOL = dict(rtol=1e-9, atol=1e-20)
ORA_TOL = dict(rtol=1e-12, atolY=1e-24, atolT=1e-9)


@pytest.fixture(scope="module")
def ora():
    return Oracle("h2air_li2004")


@pytest.fixture(scope="module")
def chem():
    return Chem("h2air_li2004", device=0, atol_T=1e-6)


def to_dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device=DEV)


def species_dev(Y, pad=0):
    """cell-major numpy [n, ns] -> component-major device [ns, n + pad] (ragged ld)."""
    n, ns = Y.shape
    out = torch.full((ns, n + pad), np.nan, dtype=torch.float64, device=DEV)
    out[:, :n] = to_dev(Y.T)
    return out


def rates_close(w_gpu, w_ora, G):
    ok = np.abs(w_gpu - w_ora) <= RTOL_RATES * G + 1e-300
    big = np.abs(w_ora) >= 1e-3 * G
    ok &= ~big | (np.abs(w_gpu - w_ora) <= RTOL_RATES * np.abs(w_ora))
    return ok


def test_structure(chem):
    assert chem.structure == "h2air_li2004"


def test_rates_parity_cfg1d(chem, ora):
    m = ora.m
    d = synth.cfg1d(m.species, m.W, n=3001)   # several tiles + a ragged tail
    Yd = species_dev(d["Y"], pad=7)
    w = chem.rates(to_dev(d["rho"]), to_dev(d["T"]), Yd).cpu().numpy()[:, :3001].T
    for i in range(3001):
        wo, qf, qr = ora.rates(d["rho"][i], d["T"][i], d["Y"][i])
        G = np.abs(m.nu_r - m.nu_f).T.astype(float) @ (np.abs(qf) + np.abs(qr))
        assert rates_close(w[i], wo, G).all(), (i, w[i], wo)


def test_rates_edge_cases(chem, ora):
    """Zero mass fractions (log 0 = -inf path), pure inert, a single species, NASA range edges."""
    m = ora.m
    ns = m.ns
    Ys, Ts = [], []
    for k in range(ns):
        y = np.zeros(ns); y[k] = 1.0
        Ys.append(y); Ts.append(1200.0)
    y = np.zeros(ns); y[0] = 0.5; y[1] = 0.5
    Ys += [y, y, y, y]
    Ts += [999.999999, 1000.0, 1000.000001, 3400.0]
    Y = np.array(Ys); T = np.array(Ts)
    rho = synth.rho_ideal(synth.P_ATM, T, Y, m.W)
    w = chem.rates(to_dev(rho), to_dev(T), species_dev(Y)).cpu().numpy().T
    for i in range(len(T)):
        wo, qf, qr = ora.rates(rho[i], T[i], Y[i])
        G = np.abs(m.nu_r - m.nu_f).T.astype(float) @ (np.abs(qf) + np.abs(qr))
        assert rates_close(w[i], wo, G).all(), i
    # pure N2: exactly zero
    assert np.all(w[ns - 1] == 0.0)


def test_energy_temperature(chem, ora):
    m = ora.m
    d = synth.cfg1d(m.species, m.W, n=1000, seed=7)
    Yd = species_dev(d["Y"])
    e = chem.energy(to_dev(d["T"]), Yd).cpu().numpy()
    eo = np.array([ora.energy(t, y) for t, y in zip(d["T"], d["Y"])])
    assert np.max(np.abs(e - eo) / np.abs(eo).clip(1e3)) < 1e-12
    T = to_dev(np.full(1000, 1500.0))
    chem.temperature(to_dev(eo), Yd, T)
    assert np.max(np.abs(T.cpu().numpy() - d["T"])) < 1e-8


def test_rhs_and_jacobian(chem, ora):
    m = ora.m
    d = synth.cfg1d(m.species, m.W, n=256, seed=9)
    Y = d["Y"] + 1e-8            # stay off the max(Y, 0) kink, where one-sided derivatives differ
    Y /= Y.sum(1, keepdims=True)
    rho, T = d["rho"], d["T"]
    f = chem.rhs(to_dev(rho), to_dev(T), species_dev(Y)).cpu().numpy()
    J = chem.jacobian(to_dev(rho), to_dev(T), species_dev(Y)).cpu().numpy()
    for i in range(len(T)):
        y = np.r_[Y[i], T[i]]
        fo = ora.rhs(rho[i], y)
        Jo = ora.jac(rho[i], y)
        wo, qf, qr = ora.rates(rho[i], T[i], Y[i])
        G = np.abs(m.nu_r - m.nu_f).T.astype(float) @ (np.abs(qf) + np.abs(qr))
        Gf = np.r_[m.W * G / rho[i], abs(fo[-1]) + 1e-300]
        assert np.all(np.abs(f[:, i] - fo) <= 1e-10 * Gf + 1e-300), i
        scale = np.abs(Jo).max(axis=1) + 1e-300
        err = np.abs(J[:, :, i] - Jo).max(axis=1) / scale
        assert err.max() < 1e-8, (i, err)


def _run_gpu(chem, rho, e, T0, Y, dt, pad=0, solid=None, **tol):
    n = len(rho)
    Td = to_dev(np.r_[T0, np.full(pad, np.nan)])[:n] if pad else to_dev(T0)
    Yd = species_dev(Y, pad)
    sd = None if solid is None else torch.as_tensor(solid, dtype=torch.uint8, device=DEV)
    st = chem.integrate(to_dev(rho), to_dev(e), Td, Yd, dt, solid=sd, **(tol or GPU_TOL))
    return Td.cpu().numpy(), Yd.cpu().numpy()[:, :n].T, st


def _check_state(T, Y, out, label):
    mask = out["Y"] > 1e-12
    relY = np.abs(Y[mask] / out["Y"][mask] - 1)
    relT = np.abs(T / out["T"] - 1)
    assert relT.max() < RTOL_STATE, (label, relT.max())
    assert relY.max() < RTOL_STATE, (label, relY.max())
    return relT.max(), relY.max()


@pytest.mark.parametrize("cfg", ["cfg1", "cfg1c"])
def test_integrate_parity(chem, ora, cfg):
    m = ora.m
    d = getattr(synth, cfg)(m.species, m.W)
    idx = np.arange(len(d["rho"])) if cfg == "cfg1" else np.arange(0, 4096, 16)   # 1c: 256 cells
    rho, T0, Y = d["rho"][idx], d["T"][idx], d["Y"][idx]
    e = np.array([ora.energy(t, y) for t, y in zip(T0, Y)])
    out = ora.integrate_cells(rho, e, T0, Y, d["dt"], **ORA_TOL)
    assert np.all(out["status"] == 0)
    T, Yg, st = _run_gpu(chem, rho, e, T0, Y, d["dt"], pad=5)
    assert st["n_unfinished"] == 0 and st["n_nonfinite"] == 0 and st["n_newton_fail"] == 0
    _check_state(T, Yg, out, cfg)


def test_gate_cold_solid_bitwise(chem, ora):
    m = ora.m
    d = synth.cfg1(m.species, m.W, n=300)
    T0 = d["T"].copy()
    T0[:50] = 300.0          # cold
    solid = np.zeros(300, dtype=np.uint8)
    solid[100:120] = 1
    e = np.array([ora.energy(t, y) for t, y in zip(T0, d["Y"])])
    Tg, Yg, st = _run_gpu(chem, d["rho"], e, T0, d["Y"], 1e-7, solid=solid)
    untouched = np.r_[np.arange(50), np.arange(100, 120)]
    assert np.array_equal(Tg[untouched], T0[untouched])
    assert np.array_equal(Yg[untouched], d["Y"][untouched])
    assert st["active0"] == 300 - 70


def test_empty_and_all_cold(chem, ora):
    m = ora.m
    st = chem.integrate(to_dev(np.zeros(0)), to_dev(np.zeros(0)), to_dev(np.zeros(0)),
                        torch.zeros((m.ns, 0), dtype=torch.float64, device=DEV), 1e-7)
    assert st["cells"] == 0
    d = synth.cfg1(m.species, m.W, n=64)
    T0 = np.full(64, 300.0)
    e = np.array([ora.energy(t, y) for t, y in zip(T0, d["Y"])])
    Tg, Yg, st = _run_gpu(chem, d["rho"], e, T0, d["Y"], 1e-7)
    assert st["active0"] == 0 and np.array_equal(Tg, T0) and np.array_equal(Yg, d["Y"])


@pytest.mark.parametrize("mech,y0,t,exact", [
    ("toy_a_to_b", [0.8, 0.2], 5e-3, lambda t: 0.8 * np.exp(-1e3 * t)),
    ("toy_a_eq_b", [0.9, 0.1], 4e-3, lambda t: 0.5 + 0.4 * np.exp(-2e3 * t)),
    ("toy_2a_to_b", [1.0, 0.0], 1e-2, lambda t: 1.0 / (1 + 2 * 10.0 * 50.0 * t)),
])
def test_closed_forms_gpu(mech, y0, t, exact):
    """SURVEY §8(c) closed forms on the CUDA path (rtol 1e-11 -> 1e-8 relative)."""
    ch = Chem(mech, device=0, atol_T=1e-9)
    o = Oracle(mech)
    n = 64
    rho = np.full(n, 1.0)
    T0 = np.full(n, 700.0)
    Y = np.tile(np.array(y0, dtype=float), (n, 1))
    e = np.array([o.energy(a, b) for a, b in zip(T0, Y)])
    Td = to_dev(T0)
    Yd = species_dev(Y)
    ch.integrate(to_dev(rho), to_dev(e), Td, Yd, t, rtol=1e-11, atol=1e-20)
    YA = Yd.cpu().numpy()[0]
    assert np.max(np.abs(YA / exact(t) - 1)) < 1e-8
    assert np.max(np.abs(Td.cpu().numpy() - 700.0)) < 1e-8


def test_schedule_invariance_bitwise(chem, ora):
    """P:177 / S:191: bulk-sparse == naive (Alg. 2) per cell, bitwise, for any K_max_bulk, N*,
    compaction mode (P:181 index map vs all-cells launches)."""
    m = ora.m
    d = synth.cfg1c(m.species, m.W)
    idx = np.arange(0, 4096, 8)
    rho, T0, Y = d["rho"][idx], d["T"][idx], d["Y"][idx]
    e = np.array([ora.energy(t, y) for t, y in zip(T0, Y)])
    ref = None
    configs = [dict(kmax_bulk=1 << 30, n_active_star=0),        # naive: one launch to t_final
               dict(kmax_bulk=1, n_active_star=0),
               dict(kmax_bulk=5, n_active_star=100),
               dict(kmax_bulk=5, n_active_star=10 ** 9),       # sparse only
               dict(kmax_bulk=3, n_active_star=50, compact_bulk=0)]
    for cfgo in configs:
        chem.set_opts(**{**dict(kmax_bulk=5, n_active_star=10000, compact_bulk=1), **cfgo})
        T, Yg, st = _run_gpu(chem, rho, e, T0, Y, d["dt"])
        # the library's own launch count: gate, a burst + compaction per bulk iteration, the sparse launch,
        # and its bookkeeping transfers (box table, counters; at least 4 of those)
        assert st["kernel_launches"] >= 1 + 2 * st["bulk_iters"] + (st["sparse_cells"] > 0) + 4, st
        if ref is None:
            ref = (T, Yg, st["steps_attempted"])
        else:
            assert np.array_equal(T, ref[0]) and np.array_equal(Yg, ref[1]), cfgo
            assert st["steps_attempted"] == ref[2]
    chem.set_opts(kmax_bulk=5, n_active_star=10000, compact_bulk=1)


def test_boxes_fused_equals_single(chem, ora):
    """A10: one fused launch over several boxes (different dt, ld) == each box alone, bitwise."""
    from paper_2510_23993_b200 import Box
    m = ora.m
    d = synth.cfg1c(m.species, m.W)
    rng = np.random.default_rng(3)
    sizes = [37, 200, 1, 64, 129]
    dts = [1e-7, 1e-5, 1e-6, 3e-5, 2e-7]
    boxes, singles = [], []
    start = 0
    for n, dt in zip(sizes, dts):
        sel = rng.integers(0, 4096, n)
        rho, T0, Y = d["rho"][sel], d["T"][sel], d["Y"][sel]
        e = np.array([ora.energy(t, y) for t, y in zip(T0, Y)])
        boxes.append(Box(to_dev(rho), to_dev(e), to_dev(T0), species_dev(Y, pad=3), dt))
        singles.append(_run_gpu(chem, rho, e, T0, Y, dt, pad=3))
        start += n
    cost = torch.zeros(len(boxes), dtype=torch.float64, device=DEV)
    st = chem.integrate_boxes(boxes, box_cost=cost, **GPU_TOL)
    for bx, (T, Yg, s1) in zip(boxes, singles):
        assert np.array_equal(bx.T.cpu().numpy(), T)
        assert np.array_equal(bx.Y.cpu().numpy()[:, :bx.ncells].T, Yg)
    c = cost.cpu().numpy()
    assert np.isclose(c.sum(), st["steps_attempted"])
    assert all(ci == s[2]["steps_attempted"] for ci, s in zip(c, singles))


def test_explicit_paper_scheme_algorithmic_parity(ora):
    """NEXT-1: the paper's explicit scheme on the CUDA path vs the oracle's step-by-step
    implementation of the same rule: identical step counts, state within 1e-10 (algorithmic parity;
    the two differ only in the rates' rounding: ln-space matrix form vs per-reaction products)."""
    import synth as _s
    doc = _s.load_trajectories()
    d = _s.cfg1b(doc, n=512)
    ch = Chem("h2air_li2004", device=0, method=2, eps_change=0.01, kmax_sparse=100000)
    e = np.array([ora.energy(t, y) for t, y in zip(d["T"], d["Y"])])
    out = ora.explicit_cells(d["rho"], e, d["T"], d["Y"], d["dt"], eps=0.01)
    assert np.all(out["status"] == 0)
    Td = to_dev(d["T"])
    Yd = species_dev(d["Y"])
    st = ch.integrate(to_dev(d["rho"]), to_dev(e), Td, Yd, d["dt"])
    assert st["n_unfinished"] == 0 and st["n_nonfinite"] == 0
    assert st["steps_attempted"] == int(out["nsteps"].sum())
    assert out["nsteps"].max() >= 10            # many explicit steps per cell
    Tg, Yg = Td.cpu().numpy(), Yd.cpu().numpy().T
    mask = out["Y"] > 1e-12
    assert np.max(np.abs(Tg / out["T"] - 1)) < 1e-10
    assert np.max(np.abs(Yg[mask] / out["Y"][mask] - 1)) < 1e-10


@pytest.mark.parametrize("cfg", ["cfg1", "cfg1c"])
def test_integrate_parity_rodas3(ora, cfg):
    """RODAS3 (CHEM_METHOD_RODAS3) reaches the same 1e-6 parity bar at the parity tolerance."""
    method = 1
    ch = Chem("h2air_li2004", device=0, atol_T=1e-6, method=method)
    m = ora.m
    d = getattr(synth, cfg)(m.species, m.W)
    idx = np.arange(0, 4096, 8) if cfg == "cfg1" else np.arange(0, 4096, 32)
    rho, T0, Y = d["rho"][idx], d["T"][idx], d["Y"][idx]
    e = np.array([ora.energy(t, y) for t, y in zip(T0, Y)])
    out = ora.integrate_cells(rho, e, T0, Y, d["dt"], **ORA_TOL)
    T, Yg, st = _run_gpu(ch, rho, e, T0, Y, d["dt"])
    assert st["n_unfinished"] == 0 and st["n_nonfinite"] == 0
    _check_state(T, Yg, out, (cfg, method))


def test_fault_injection_counts(ora):
    """SPEC S:184 / SURVEY §5: per-cell problems are counts, not call errors.  A tiny K_max_sparse
    leaves cells unfinished (state at the last accepted step); NaN inputs are counted and do not
    disturb the other cells; T far outside the NASA ranges is extrapolated and counted."""
    m = ora.m
    d = synth.cfg1c(m.species, m.W)
    idx = np.arange(0, 4096, 64)
    rho, T0, Y = d["rho"][idx].copy(), d["T"][idx].copy(), d["Y"][idx].copy()
    e = np.array([ora.energy(t, y) for t, y in zip(T0, Y)])
    ch = Chem("h2air_li2004", device=0, kmax_bulk=2, n_active_star=10 ** 9, kmax_sparse=3)
    T, Yg, st = _run_gpu(ch, rho, e, T0, Y, d["dt"])
    assert st["n_unfinished"] > 0 and st["n_nonfinite"] == 0
    assert np.all(np.isfinite(T)) and np.all(np.isfinite(Yg))
    # the per-cell status output names exactly the counted cells
    status = ch.cell_status().cpu().numpy()
    assert len(status) == len(rho)
    assert (status == 2).sum() == st["n_unfinished"] and set(np.unique(status)) <= {1, 2}
    # NaN in one cell's Y: counted as a failure, neighbours bitwise equal to a clean run
    ch2 = Chem("h2air_li2004", device=0)
    Tc, Yc, _ = _run_gpu(ch2, rho, e, T0, Y, 1e-7)
    Yb = Y.copy()
    Yb[5, 3] = np.nan
    Tn, Yn, st2 = _run_gpu(ch2, rho, e, T0, Yb, 1e-7)
    assert st2["n_nonfinite"] + st2["n_newton_fail"] >= 1
    status2 = ch2.cell_status().cpu().numpy()
    assert status2[5] == -1 and np.all(np.delete(status2, 5) == 1)
    keep = np.arange(len(rho)) != 5
    assert np.array_equal(Tn[keep], Tc[keep]) and np.array_equal(Yn[keep], Yc[keep])
    # very hot cell: beyond the 3500 K NASA range -> counted in n_T_range, still finite
    Th = np.full(4, 3200.0)
    Yh = np.tile(d["Y"][0], (4, 1))
    rh = synth.rho_ideal(synth.P_ATM * 30, Th, Yh, m.W)
    eh = np.array([ora.energy(t, y) for t, y in zip(Th, Yh)])
    Tg, Yg2, st3 = _run_gpu(ch2, rh, eh, Th, Yh, 1e-5)
    assert np.all(np.isfinite(Tg)) and st3["n_T_range"] >= 1 and st3["n_unfinished"] == 0


def test_invalid_arguments_are_errors():
    from paper_2510_23993_b200.binding import ChemError
    ch = Chem("h2air_li2004", device=0)
    z = torch.zeros(4, dtype=torch.float64, device=DEV)
    Y = torch.zeros((9, 4), dtype=torch.float64, device=DEV)
    with pytest.raises(ChemError):
        ch.integrate(z, z, z.clone(), Y, dt=-1.0)
    with pytest.raises(ChemError):
        ch.integrate(z, z, z.clone(), Y, dt=1e-7, rtol=0.0)
    with pytest.raises(ChemError):
        ch.set_opts(kmax_bulk=0)
    with pytest.raises(TypeError):
        ch.integrate(z.cpu(), z, z.clone(), Y, 1e-7)
    # the binding guards what the C ABI cannot see: short, float32, foreign-device or
    # mis-shaped buffers, a short box_cost, unknown option names
    with pytest.raises(ValueError):
        ch.integrate(z, z, z[:3].clone(), Y, 1e-7)
    with pytest.raises(TypeError):
        ch.integrate(z, z.float(), z.clone(), Y, 1e-7)
    with pytest.raises(ValueError):
        ch.integrate(z, z, z.clone(), Y[:, :3], 1e-7)
    from paper_2510_23993_b200 import Box
    with pytest.raises(ValueError):
        ch.integrate_boxes([Box(z, z, z.clone(), Y, 1e-7)] * 2,
                           box_cost=torch.zeros(1, dtype=torch.float64, device=DEV))
    with pytest.raises(TypeError):
        ch.set_opts(lanes_per_cell=4)


def test_internal_energy_alg1():
    """NEXT-4 / PAPER.md Alg. 1: e = rho E/rho - |u|^2/2, element by element (the definition)."""
    ch = Chem("h2air_li2004", device=0)
    rng = np.random.default_rng(4)
    n = 1000
    rho = rng.uniform(0.1, 5.0, n)
    u = rng.normal(0, 800.0, (3, n))
    eint = rng.uniform(1e5, 3e6, n)
    E = eint + 0.5 * (u ** 2).sum(0)
    U = np.vstack([rho, rho * u[0], rho * u[1], rho * u[2], rho * E])
    Ud = torch.zeros((5, n + 3), dtype=torch.float64, device=DEV)
    Ud[:, :n] = to_dev(U)
    e = ch.internal_energy(Ud)[:n].cpu().numpy()
    assert np.max(np.abs(e / eint - 1)) < 1e-12


def test_strang_half_steps_equal_full_step(ora):
    """Two chemistry half steps (Strang, with a frozen flow in between) reproduce one
    integration over the full dt to the parity tolerance."""
    from paper_2510_23993_b200 import Box
    m = ora.m
    d = synth.cfg1c(m.species, m.W)
    idx = np.arange(0, 4096, 128)
    rho, T0, Y = d["rho"][idx], d["T"][idx], d["Y"][idx]
    e = np.array([ora.energy(t, y) for t, y in zip(T0, Y)])
    ch = Chem("h2air_li2004", device=0, atol_T=1e-6)
    box = Box(to_dev(rho), to_dev(e), to_dev(T0), species_dev(Y), 0.0)
    ch.strang_half_step([box], 2e-5, **GPU_TOL)
    ch.strang_half_step([box], 2e-5, **GPU_TOL)
    out = ora.integrate_cells(rho, e, T0, Y, 2e-5, **ORA_TOL)
    _check_state(box.T.cpu().numpy(), box.Y.cpu().numpy().T, out, "strang")


def test_cgs_toy_closed_forms_gpu():
    """VERDICT r01 next-1a on the CUDA path: mech/toy_cgs_falloff.yaml (cm/mol/cal units) through the
    product loader and the kernels against tests/pins/cgs_toy.py's hand-converted SI closed forms:
    rates at t = 0 (1e-12) and the integrated three-body / Lindemann / Troe / second-order decays
    (rtol 1e-11 -> 1e-8), isothermal at 1000 K."""
    from tests.pins import cgs_toy as ct
    ch = Chem("toy_cgs_falloff", device=0, atol_T=1e-9)
    sp = ch.mech.species.index
    rho = ct.rho_at_troe_centre()
    n = 40
    Y = np.zeros((n, ch.ns))
    for k, v in ct.Y0.items():
        Y[:, sp(k)] = v
    lam1, lam2, lam3, k4 = ct.decay_rates(rho)
    c = rho * Y[0] / ct.W
    w = ch.rates(to_dev(np.full(n, rho)), to_dev(np.full(n, ct.T)), species_dev(Y)).cpu().numpy()[:, 0]
    for name, v in (("A1", -lam1 * c[sp("A1")]), ("A2", -lam2 * c[sp("A2")]), ("A3", -lam3 * c[sp("A3")]),
                    ("A4", -2.0 * k4 * c[sp("A4")] ** 2)):
        assert abs(w[sp(name)] / v - 1) < 1e-12, (name, w[sp(name)], v)
    o = Oracle("toy_cgs_falloff")
    e = np.full(n, o.energy(ct.T, Y[0]))
    t = 1e-5
    Td = to_dev(np.full(n, ct.T))
    Yd = species_dev(Y)
    st = ch.integrate(to_dev(np.full(n, rho)), to_dev(e), Td, Yd, t, rtol=1e-11, atol=1e-20)
    assert st["n_unfinished"] == 0
    Yg = Yd.cpu().numpy()
    for name, v in zip(("A1", "A2", "A3", "A4"), ct.exact_Y(rho, t)):
        assert np.max(np.abs(Yg[sp(name)] / v - 1)) < 1e-8, name
    assert np.max(np.abs(Td.cpu().numpy() - ct.T)) < 1e-8


def test_negative_Y_edge(chem, ora):
    """SURVEY reading 5 at the kink: rates use max(Y, 0) and the Jacobian column of a species with
    Y < 0 is zero (cj = 0), on both sides; integrating from slightly negative radicals (the
    integrator's own output, |Y| <= atol) stays within the parity bar."""
    m = ora.m
    d = synth.cfg1d(m.species, m.W, n=128, seed=11)
    Y = d["Y"].copy()
    rng = np.random.default_rng(12)
    neg = rng.random(Y.shape) < 0.15
    neg[:, m.species.index("N2")] = False
    Y[neg] = -rng.uniform(1e-22, 1e-12, neg.sum())
    rho, T = d["rho"], d["T"]
    w = chem.rates(to_dev(rho), to_dev(T), species_dev(Y)).cpu().numpy()
    J = chem.jacobian(to_dev(rho), to_dev(T), species_dev(Y)).cpu().numpy()
    for i in range(len(T)):
        wo, qf, qr = ora.rates(rho[i], T[i], Y[i])
        G = np.abs(m.nu_r - m.nu_f).T.astype(float) @ (np.abs(qf) + np.abs(qr))
        assert rates_close(w[:, i], wo, G).all(), i
        Jo = ora.jac(rho[i], np.r_[Y[i], T[i]])
        for k in np.nonzero(neg[i])[0]:
            assert np.all(J[:m.ns, k, i] == 0.0), (i, k)      # the species block column is zero
        scale = np.abs(Jo).max(axis=1) + 1e-300
        assert (np.abs(J[:, :, i] - Jo).max(axis=1) / scale).max() < 1e-8, i
    # integration from a radical-rich state with tiny negative radicals
    doc = synth.load_trajectories()
    d1 = synth.cfg1b(doc, n=256)
    Y1 = d1["Y"].copy()
    for k in ("H", "O", "HO2", "H2O2"):
        Y1[::3, m.species.index(k)] = -1e-21
    e1 = np.array([ora.energy(t, y) for t, y in zip(d1["T"], Y1)])
    out = ora.integrate_cells(d1["rho"], e1, d1["T"], Y1, d1["dt"], **ORA_TOL)
    assert np.all(out["status"] == 0)
    Tg, Yg, st = _run_gpu(chem, d1["rho"], e1, d1["T"], Y1, d1["dt"])
    assert st["n_nonfinite"] == 0 and st["n_unfinished"] == 0
    _check_state(Tg, Yg, out, "negative-Y")


def test_budget_equivalence_lpt_vs_alg3(ora):
    """kmax_sparse is the per-cell budget of attempted substeps over the whole
    call, so a cell that hits it ends UNFINISHED in the same state under Alg. 3 (bulk bursts +
    sparse launch) and under the heavy-first launch: bitwise equal outputs, statuses and counts."""
    m = ora.m
    d = synth.cfg1c(m.species, m.W)
    idx = np.arange(0, 4096, 16)
    rho, T0, Y = d["rho"][idx], d["T"][idx], d["Y"][idx]
    e = np.array([ora.energy(t, y) for t, y in zip(T0, Y)])
    res = []
    for opts in (dict(schedule_lpt=0, kmax_bulk=5, n_active_star=0),
                 dict(schedule_lpt=0, kmax_bulk=3, n_active_star=64),
                 dict(schedule_lpt=1), dict(schedule_lpt=0, n_active_star=10 ** 9),
                 dict(schedule_lpt=3, kmax_bulk=2, n_active_star=0)):
        ch = Chem("h2air_li2004", device=0, kmax_sparse=12, **opts)
        _run_gpu(ch, rho, e, T0, Y, d["dt"])        # leaves cost hints (the heavy-first launch needs them)
        T, Yg, st = _run_gpu(ch, rho, e, T0, Y, d["dt"])
        assert st["lpt"] == {1: 1, 3: 2}.get(opts.get("schedule_lpt"), 0), (opts, st["lpt"])
        res.append((T, Yg, ch.cell_status().cpu().numpy(), st["n_unfinished"], st["steps_attempted"]))
    assert res[0][3] > 0
    for r in res[1:]:
        assert np.array_equal(r[0], res[0][0]) and np.array_equal(r[1], res[0][1])
        assert np.array_equal(r[2], res[0][2]) and r[3:] == res[0][3:]


def test_cell_status_multibox_and_box_active(ora):
    """chem_cell_status numbers the cells of a fused call box after box; chem_box_active counts what the
    gate would integrate per box without touching the workspace; forget_hints clears the cost hints."""
    from paper_2510_23993_b200 import Box
    m = ora.m
    d = synth.cfg1(m.species, m.W, n=300)
    T0 = d["T"].copy()
    T0[:100] = 300.0                                   # box 0 entirely cold
    e = np.array([ora.energy(t, y) for t, y in zip(T0, d["Y"])])
    ch = Chem("h2air_li2004", device=0, kmax_sparse=4)
    solid = torch.zeros(100, dtype=torch.uint8, device=DEV)
    solid[:10] = 1
    boxes = [Box(to_dev(d["rho"][a:b]), to_dev(e[a:b]), to_dev(T0[a:b]), species_dev(d["Y"][a:b]), 1e-6,
                 solid if a == 200 else None) for a, b in ((0, 100), (100, 200), (200, 300))]
    act = ch.box_active(boxes).cpu().tolist()
    assert act == [0, 100, 90]
    st = ch.integrate_boxes(boxes, rtol=1e-9, atol=1e-20)
    status, steps = ch.cell_status(substeps=True)
    status, steps = status.cpu().numpy(), steps.cpu().numpy()
    assert len(status) == 300 and st["active0"] == 190
    assert np.all(status[:100] == 0) and np.all(status[200:210] == 0) and np.all(steps[:100] == 0)
    assert set(np.unique(status[100:200])) <= {1, 2} and set(np.unique(status[210:])) <= {1, 2}
    assert (status == 2).sum() == st["n_unfinished"]
    assert int(steps.sum()) == st["steps_attempted"]
    part = ch.cell_status(n=50, first=150).cpu().numpy()
    assert np.array_equal(part, status[150:200])
    with pytest.raises(Exception):
        ch.cell_status(n=10, first=295)                # beyond the call's cells
    ch.forget_hints()
    st2 = ch.integrate_boxes(boxes, rtol=1e-9, atol=1e-20)
    assert st2["hint_accuracy"] == -1.0               # no hints after forget_hints

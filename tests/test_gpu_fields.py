"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times (fused
chem_integrate_boxes over every box, default schedule, parity tolerance): sampled cells against the
oracle one by one, plus properties that hold at any size (cold cells bitwise untouched, identical
inputs -> bitwise identical outputs, no unfinished/failed cells).

Each side evaluates e = u(T0, Y) with its own thermo (no oracle input comes from the CUDA path)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import Oracle  # noqa: E402
from paper_2510_23993_b200 import Box, Chem  # noqa: E402

DEV = torch.device("cuda", 0)
GPU_TOL = dict(rtol=1e-9, atol=1e-20)
ORA_TOL = dict(rtol=1e-12, atolY=1e-24, atolT=1e-9)
REL = 1e-6


@pytest.fixture(scope="module")
def ora():
    return Oracle("h2air_li2004")


@pytest.fixture(scope="module")
def chem():
    return Chem("h2air_li2004", device=0, atol_T=1e-6)


@pytest.fixture(scope="module")
def doc():
    return synth.load_trajectories()


def _run(chem, raw):
    boxes = []
    for b in raw:
        e = chem.energy(b["T"], b["Y"])
        boxes.append(Box(b["rho"], e, b["T"].clone(), b["Y"].clone(), b["dt"], b.get("solid")))
    cost = torch.zeros(len(boxes), dtype=torch.float64, device=DEV)
    st = chem.integrate_boxes(boxes, box_cost=cost, **GPU_TOL)
    torch.cuda.synchronize()
    return boxes, st, cost


def _sample_and_check(ora, raw, boxes, picks):
    """picks: list of (box index, cell offset).  Oracle on the sampled inputs, compare outputs."""
    rho = np.array([raw[b]["rho"][i].item() for b, i in picks])
    T0 = np.array([raw[b]["T"][i].item() for b, i in picks])
    Y0 = np.array([raw[b]["Y"][:, i].cpu().numpy() for b, i in picks])
    dt = np.array([raw[b]["dt"] for b, i in picks])
    e = np.array([ora.energy(t, y) for t, y in zip(T0, Y0)])
    worst = (0.0, 0.0)
    for d in np.unique(dt):
        sel = dt == d
        out = ora.integrate_cells(rho[sel], e[sel], T0[sel], Y0[sel], float(d), **ORA_TOL)
        assert np.all(out["status"] >= 0)
        for q, (b, i) in enumerate([p for p, s in zip(picks, sel) if s]):
            Tg = boxes[b].T[i].item()
            Yg = boxes[b].Y[:, i].cpu().numpy()
            if out["status"][q] == 1:      # gated: bitwise untouched
                assert Tg == T0[sel][q] and np.array_equal(Yg, Y0[sel][q])
                continue
            mask = out["Y"][q] > 1e-12
            rT = abs(Tg / out["T"][q] - 1)
            rY = np.max(np.abs(Yg[mask] / out["Y"][q][mask] - 1))
            worst = (max(worst[0], rT), max(worst[1], rY))
            assert rT < REL and rY < REL, (b, i, rT, rY)
    return worst


def _cold_untouched(raw, boxes, T_min=500.0):
    for r, b in zip(raw, boxes):
        cold = r["T"] < T_min
        assert torch.equal(b.T[cold], r["T"][cold])
        assert torch.equal(b.Y[:, cold], r["Y"][:, cold])


def test_cfg1b_radical_rich(chem, ora, doc):
    d = synth.cfg1b(doc, n=2048)
    e = np.array([ora.energy(t, y) for t, y in zip(d["T"], d["Y"])])
    out = ora.integrate_cells(d["rho"], e, d["T"], d["Y"], d["dt"], **ORA_TOL)
    Td = torch.tensor(d["T"], device=DEV)
    Yd = torch.tensor(d["Y"].T.copy(), device=DEV)
    st = chem.integrate(torch.tensor(d["rho"], device=DEV), torch.tensor(e, device=DEV), Td, Yd, d["dt"], **GPU_TOL)
    assert st["n_unfinished"] == 0 and st["n_nonfinite"] == 0
    Tg, Yg = Td.cpu().numpy(), Yd.cpu().numpy().T
    mask = out["Y"] > 1e-12
    assert np.max(np.abs(Tg / out["T"] - 1)) < REL
    assert np.max(np.abs(Yg[mask] / out["Y"][mask] - 1)) < REL


def test_cfg2_full_size(chem, ora, doc):
    raw, meta = synth.field_cfg2(doc, device=DEV)
    boxes, st, cost = _run(chem, raw)
    assert st["cells"] == 128 ** 3 and st["active0"] == 128 ** 3
    assert st["n_unfinished"] == 0 and st["n_nonfinite"] == 0
    # identical inputs -> bitwise identical outputs (any size)
    for b in boxes:
        assert torch.all(b.T == boxes[0].T[0]) and torch.all(b.Y == boxes[0].Y[:, :1])
    rng = np.random.default_rng(0)
    picks = [(int(rng.integers(0, 64)), int(rng.integers(0, 32 ** 3))) for _ in range(16)]
    _sample_and_check(ora, raw, boxes, picks)
    c = cost.cpu().numpy()
    assert np.allclose(c, c[0]) and np.isclose(c.sum(), st["steps_attempted"])


@pytest.mark.parametrize("lanes", [1, 8])
def test_cfg3_full_size(ora, doc, lanes):
    chem = Chem("h2air_li2004", device=0, atol_T=1e-6, lanes_per_cell=lanes)
    m = ora.m
    raw, meta = synth.field_cfg3(doc, m.W, m.species, device=DEV)
    n_act = sum(int((r["T"] >= 500).sum()) for r in raw)
    boxes, st, cost = _run(chem, raw)
    assert st["cells"] == 256 ** 3 and st["active0"] == n_act
    assert 0.01 < n_act / 256 ** 3 < 0.03          # ~2% active (BASELINE configs[2])
    assert st["n_unfinished"] == 0 and st["n_nonfinite"] == 0
    _cold_untouched(raw, boxes)
    rng = np.random.default_rng(1)
    picks = []
    for b, r in enumerate(raw):
        act = torch.nonzero(r["T"] >= 500).flatten().cpu().numpy()
        if len(act):
            picks += [(b, int(i)) for i in rng.choice(act, size=min(4, len(act)), replace=False)]
    picks += [(0, 64 * 64 * 32 + 40)]                 # one cold cell
    _sample_and_check(ora, raw, boxes, picks)


def test_cfg4_one_copy_all_levels_fused(chem, ora, doc):
    m = ora.m
    descs = synth.hierarchy_cfg4(copy=1)
    raw = [synth.build_cfg4_box(doc, m.W, m.species, d, DEV) for d in descs]
    boxes, st, cost = _run(chem, raw)               # three levels, three dt, one fused launch per phase
    assert st["cells"] == 192 * 32 ** 3
    assert st["n_unfinished"] == 0 and st["n_nonfinite"] == 0
    _cold_untouched(raw, boxes)
    rng = np.random.default_rng(2)
    picks = []
    for b in rng.choice(len(raw), size=24, replace=False):
        act = torch.nonzero(raw[b]["T"] >= 500).flatten().cpu().numpy()
        if len(act):
            picks.append((int(b), int(rng.choice(act))))
    _sample_and_check(ora, raw, boxes, picks)


def test_cfg5_rank_shard(chem, ora, doc):
    """One GPU's share of the 8-GPU jet-in-crossflow field (16 of 128 boxes around the jet)."""
    m = ora.m
    ids = [1, 2, 9, 10, 17, 18, 25, 26, 41, 42, 49, 50, 57, 58, 3, 11]
    raw, meta = synth.field_cfg5(doc, m.W, m.species, device=DEV, box_ids=ids)
    boxes, st, cost = _run(chem, raw)
    assert st["n_unfinished"] == 0 and st["n_nonfinite"] == 0
    _cold_untouched(raw, boxes)
    rng = np.random.default_rng(3)
    picks = []
    for b, r in enumerate(raw):
        shear = torch.nonzero((r["T"] >= 900) & (r["Y"][0] > 1e-3)).flatten().cpu().numpy()
        hot = torch.nonzero(r["T"] >= 500).flatten().cpu().numpy()
        for pool in (shear, hot):
            if len(pool):
                picks.append((b, int(rng.choice(pool))))
    _sample_and_check(ora, raw, boxes, picks)


def test_virtual_ranks_bitwise(chem, ora, doc):
    """per-cell results do not depend on the box -> rank map.  One copy of the
    cfg4 hierarchy integrated as one fused call equals the same boxes split over 'virtual ranks'
    (LPT on their measured cost, each rank's boxes in its own fused call), bitwise."""
    from paper_2510_23993_b200.sharding import lpt_partition
    m = ora.m
    descs = [d for d in synth.hierarchy_cfg4(copy=2) if d["index"] % 4 == 0]     # 48 boxes, 3 levels
    raw = [synth.build_cfg4_box(doc, m.W, m.species, d, DEV) for d in descs]
    whole, st, cost = _run(chem, raw)
    owner = lpt_partition(cost.cpu().numpy(), 3)
    for r in range(3):
        mine = [i for i in range(len(raw)) if owner[i] == r]
        if not mine:
            continue
        part, _, _ = _run(chem, [raw[i] for i in mine])
        for j, i in enumerate(mine):
            assert torch.equal(part[j].T, whole[i].T) and torch.equal(part[j].Y, whole[i].Y)


@pytest.mark.parametrize("opts", [dict(refill_bulk=1), dict(kmax_bulk=20, n_active_star=3000),
                                  dict(compact_bulk=0, kmax_bulk=3), dict(lockstep=1),
                                  dict(lockstep=1, kmax_first=0, kmax_bulk=3), dict(lockstep=1, compact_bulk=0),
                                  dict(lockstep_sparse=1), dict(schedule_lpt=1)])
def test_cfg3_schedule_variants_bitwise(ora, doc, opts):
    """Bulk-sparse variants (lane-refill bursts, longer bursts, the paper's all-cells bursts) give
    bitwise the same field as the default schedule (P:177 / S:191), at full cfg3 size."""
    m = ora.m
    ids = [0, 16, 32, 48]                    # the four boxes along y at x = 0 (band + spots)
    raw, _ = synth.field_cfg3(doc, m.W, m.species, device=DEV, box_ids=ids)
    ref, st0, _ = _run(Chem("h2air_li2004", device=0, atol_T=1e-6, lockstep=0, schedule_lpt=0), raw)
    alt, st1, _ = _run(Chem("h2air_li2004", device=0, atol_T=1e-6, **opts), raw)
    assert st1["lockstep"] == opts.get("lockstep", 0)
    for a, b in zip(ref, alt):
        assert torch.equal(a.T, b.T) and torch.equal(a.Y, b.Y)
    assert st0["steps_attempted"] == st1["steps_attempted"]


def test_activity_trace_app_b(ora, doc):
    """App. B instrumentation: per-box active counts after the gate and each bulk launch,
    consistent with the gate count and the per-iteration totals; App. B line format."""
    from paper_2510_23993_b200.api import activity_lines
    m = ora.m
    raw, _ = synth.field_cfg3(doc, m.W, m.species, device=DEV, box_ids=[0, 1, 16, 17])
    ch = Chem("h2air_li2004", device=0, atol_T=1e-6, n_active_star=100)
    tr = ch.set_trace(12, len(raw))
    boxes, st, _ = _run(ch, raw)
    t = tr.cpu().numpy()
    for b, r in enumerate(raw):
        assert t[0, b] == int((r["T"] >= 500).sum())
    for i in range(1, min(12, st["bulk_iters"] + 1)):
        assert t[i].sum() == st["active_per_iter"][i - 1]
        assert np.all(t[i] <= t[i - 1])
    lines = activity_lines(tr, boxes, t=1e-7, kmax=5)
    assert lines[0].startswith("Level 0, FAB 0, t = 1e-07, step = 0, n_cells = 262144, n_active = ")
    ch.set_trace(0, 0)


@pytest.mark.parametrize("chunks", [1, 3])
def test_host_runner_matches_device_path(chem, doc, chunks):
    """The e2e path (HostRunner: pinned slabs, one H2D and one D2H copy per group, copy/compute
    pipelining) returns bitwise the same (T, Y) as the device-resident call on the same boxes."""
    from paper_2510_23993_b200.api import HostRunner
    rng = np.random.default_rng(5)
    d = synth.cfg1b(doc, n=6 * 512)
    host, dev_boxes = [], []
    for b in range(6):
        sl = slice(b * 512, (b + 1) * 512)
        T = torch.tensor(d["T"][sl], dtype=torch.float64)
        Y = torch.tensor(d["Y"][sl].T.copy(), dtype=torch.float64)
        rho = torch.tensor(d["rho"][sl], dtype=torch.float64)
        e = chem.energy(T.to(DEV), Y.to(DEV)).cpu()
        host.append(dict(rho=rho.pin_memory(), e=e.pin_memory(), T=T.pin_memory(), Y=Y.pin_memory(), dt=d["dt"]))
        dev_boxes.append(Box(rho.to(DEV), e.to(DEV), T.to(DEV), Y.to(DEV), d["dt"]))
    chem.integrate_boxes(dev_boxes, **GPU_TOL)
    hr = HostRunner(chem, host, chunks=chunks)
    assert hr.pipelined == (chunks > 1)
    for _ in range(2):                                   # a second step starts from the same inputs
        hr.step(**GPU_TOL)
        torch.cuda.synchronize()
        for i, b in enumerate(dev_boxes):
            assert torch.equal(hr.out_T[i], b.T.cpu()) and torch.equal(hr.out_Y[i], b.Y.cpu())
    assert hr.h2d_bytes == 6 * 512 * (3 + len(doc["species"])) * 8
    assert hr.d2h_bytes == 6 * 512 * (1 + len(doc["species"])) * 8
    del rng


def test_cfg3_heavy_first_second_call_bitwise(ora, doc):
    """Heavy-first schedule (schedule_lpt = 2): the second call on the same layout sorts the active list
    by the first call's per-cell substeps and runs it as one persistent lockstep launch (the first
    call may or may not find hints: a recycled workspace block can carry a signature of the same
    layout).  Every call gives bitwise the default schedule's field."""
    m = ora.m
    ids = [0, 16, 32, 48]
    raw, _ = synth.field_cfg3(doc, m.W, m.species, device=DEV, box_ids=ids)
    ref, st0, _ = _run(Chem("h2air_li2004", device=0, atol_T=1e-6, schedule_lpt=0), raw)
    chem = Chem("h2air_li2004", device=0, atol_T=1e-6, schedule_lpt=2)
    boxes = []
    for b in raw:
        e = chem.energy(b["T"], b["Y"])
        boxes.append(Box(b["rho"], e, b["T"].clone(), b["Y"].clone(), b["dt"], b.get("solid")))
    for call in range(2):
        for bx, b in zip(boxes, raw):
            bx.T.copy_(b["T"])
            bx.Y.copy_(b["Y"])
        st = chem.integrate_boxes(boxes, **GPU_TOL)
        torch.cuda.synchronize()
        if call == 1:
            assert st["lpt"] == 1                      # the first call left hints for this layout
        assert st["steps_attempted"] == st0["steps_attempted"]
        for a, b in zip(ref, boxes):
            assert torch.equal(a.T, b.T) and torch.equal(a.Y, b.Y)

"""Pins for the oracle's implementation of the paper's explicit scheme (SPEC.md
S:127-144, NEXT-1): the adaptive-dt examples of S:133-135, the frozen case of S:142, the first-order
convergence of S:143 against the closed form Y_A = exp(-k t), and energy conservation."""
import numpy as np

from oracle import Oracle


def test_adaptive_dt_rule_toy():
    """S:133 (dt = eps * Y/|dY/dt|): A->B, k = 1e3, Y0 = (0.5, 0.5).  A limits every step
    (Y_A/|dY_A/dt| = 1/k; B's ratio Y_B/(k Y_A) >= 1/k since Y_B >= Y_A), so dt = eps/k = 1e-5 s,
    t = 1e-4 takes exactly 10 steps and Y_A = 0.5 (1 - eps)^10."""
    o = Oracle("toy_a_to_b")
    r = o.explicit_cells(np.array([1.0]), np.array([o.energy(600.0, [0.5, 0.5])]), np.array([600.0]),
                         np.array([[0.5, 0.5]]), 1e-4, eps=0.01)
    assert r["status"][0] == 0 and r["nsteps"][0] == 10
    assert abs(r["Y"][0, 0] - 0.5 * 0.99 ** 10) < 1e-14


def test_remaining_time_caps_dt():
    """remaining time smaller than the rate-limited step -> one step of the remaining time."""
    o = Oracle("toy_a_to_b")
    r = o.explicit_cells(np.array([1.0]), np.array([o.energy(600.0, [1.0, 0.0])]), np.array([600.0]),
                         np.array([[1.0, 0.0]]), 1e-6, eps=0.01)
    assert r["nsteps"][0] == 1
    assert abs(r["Y"][0, 0] - (1.0 - 1e3 * 1e-6)) < 1e-15


def test_frozen_one_step(oracle_h2):
    """S:134 / S:142: all rates zero (pure N2) -> one step of the whole interval, Y unchanged."""
    o = oracle_h2
    Y = np.zeros(9); Y[-1] = 1.0
    T0 = 1500.0
    r = o.explicit_cells(np.array([0.3]), np.array([o.energy(T0, Y)]), np.array([T0]), Y[None], 1e-4)
    assert r["nsteps"][0] == 1 and np.array_equal(r["Y"][0], Y) and abs(r["T"][0] - T0) < 1e-9


def test_first_order_convergence():
    """final-Y error vs exp(-k t) scales ~O(eps): halving eps halves the error (factor 1.5-3)."""
    o = Oracle("toy_a_to_b")
    errs = []
    for eps in (0.04, 0.02, 0.01):
        r = o.explicit_cells(np.array([1.0]), np.array([o.energy(600.0, [1.0, 0.0])]), np.array([600.0]),
                             np.array([[1.0, 0.0]]), 2e-3, eps=eps)
        errs.append(abs(r["Y"][0, 0] - np.exp(-2.0)))
    for a, b in zip(errs, errs[1:]):
        assert 1.5 <= a / b <= 3.0, errs


def test_energy_conserved_and_clip(oracle_h2):
    """e(T_out, Y_out) equals e_in to the Newton tolerance; Y never negative (clip)."""
    o = oracle_h2
    m = o.m
    X = np.zeros(9); X[0], X[1], X[-1] = 2.0, 1.0, 3.76
    Y0 = X * m.W / np.sum(X * m.W)
    Y0[3] = 1e-6; Y0 /= Y0.sum()             # seed some H radicals so the tail is active
    T0 = 1400.0
    rho = 101325.0 / (8.314462618 * T0 * np.sum(Y0 / m.W))
    e = o.energy(T0, Y0)
    r = o.explicit_cells(np.array([rho]), np.array([e]), np.array([T0]), Y0[None], 2e-5)
    assert r["status"][0] == 0 and r["nsteps"][0] > 50          # the long explicit tail
    assert np.all(r["Y"][0] >= 0.0)
    assert abs(o.energy(r["T"][0], r["Y"][0]) / e - 1) < 1e-12
    assert r["T"][0] > T0 + 100                                 # it ignited

"""Pin the Rosenbrock coefficients compiled into the CUDA path (csrc/chem_device.cuh) against the
Rosenbrock order conditions (Hairer & Wanner, Solving ODEs II, Sec. IV.7, Table 7.1), in the
transformed form (I/(h gamma) - J) K_i = f(y + sum a_ij K_j) + sum (c_ij/h) K_j, y1 = y + sum m_j K_j:
Gamma^{-1} = I/gamma - C, alpha = A Gamma, b = m Gamma.  A mistyped digit breaks a condition."""
import pathlib
import re

import numpy as np
import pytest

SRC = (pathlib.Path(__file__).resolve().parent.parent / "paper_2510_23993_b200" / "csrc" / "chem_device.cuh").read_text()


def _table(name):
    m = re.search(name + r"\[(\d+)\]\[(\d+)\] = \{(.*?)\};", SRC, re.S)
    rows = re.findall(r"\{([^{}]*)\}", m.group(3))
    return np.array([[eval(x) for x in r.split(",")] for r in rows], dtype=float)


def _m_vector(struct):
    body = SRC[SRC.index(f"struct {struct} {{"):]
    m = re.search(r"constexpr double t\[\d+\] = \{([^}]*)\};\s*return t\[i\];", body[body.index("m(int i)"):])
    return np.array([eval(x) for x in m.group(1).split(",")], dtype=float)


def _conditions(A, C, m, gamma):
    s = len(m)
    G = np.linalg.inv(np.eye(s) / gamma - C)
    alpha = A @ G
    b = m @ G
    beta = np.tril(alpha + G, -1)
    bp = beta.sum(1)
    a = alpha.sum(1)
    return np.array([
        b.sum() - 1,
        b @ bp - (0.5 - gamma),
        b @ a ** 2 - 1 / 3,
        b @ (beta @ bp) - (1 / 6 - gamma + gamma ** 2),
        b @ a ** 3 - 1 / 4,
        b @ (a * (alpha @ bp)) - (1 / 8 - gamma / 3),
        b @ (beta @ a ** 2) - (1 / 12 - gamma / 3),
        b @ (beta @ (beta @ bp)) - (1 / 24 - gamma / 2 + 1.5 * gamma ** 2 - gamma ** 3),
    ]), alpha


def _e_vector(struct, s):
    body = SRC[SRC.index(f"struct {struct} {{"):]
    ebody = body[body.index("e(int i)"):][:400]
    m = re.search(r"constexpr double t\[\d+\] = \{([^}]*)\};", ebody)
    if m:
        return np.array([eval(x) for x in m.group(1).split(",")], dtype=float)
    e = np.zeros(s); e[-1] = 1.0          # "return i == S-1 ? 1 : 0"
    return e


@pytest.mark.parametrize("struct,Aname,Cname,gamma,order", [("Rodas4", "kRodas4A", "kRodas4C", 0.25, 4),
                                                          ("Rodas3", "kRodas3A", "kRodas3C", 0.5, 3)])
def test_order_conditions(struct, Aname, Cname, gamma, order):
    A, C, m = _table(Aname), _table(Cname), _m_vector(struct)
    res, alpha = _conditions(A, C, m, gamma)
    nconds = {3: 4, 4: 8}[order]
    assert np.max(np.abs(res[:nconds])) < 1e-13, res
    # embedded method (m - e, e = last stage) is one order lower
    e = _e_vector(struct, len(m))
    res_e, _ = _conditions(A, C, m - e, gamma)
    nlow = {3: 2, 4: 4}[order]
    assert np.max(np.abs(res_e[:nlow])) < 1e-13
    assert np.max(np.abs(res_e[nlow:nconds])) > 1e-4        # and genuinely lower order
    if struct == "Rodas4":
        assert np.allclose(alpha.sum(1)[1:4], [0.386, 0.21, 0.63], atol=1e-13)   # c_i of RODAS4


def test_stiff_accuracy_rodas4():
    """Stiffly accurate: the last stage's abscissa is 1 (alpha row sums of stages 5, 6 equal 1)."""
    A, C, m = _table("kRodas4A"), _table("kRodas4C"), _m_vector("Rodas4")
    _, alpha = _conditions(A, C, m, 0.25)
    assert np.allclose(alpha.sum(1)[4:], 1.0, atol=1e-13)

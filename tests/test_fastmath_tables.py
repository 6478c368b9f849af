"""The exp/log tables of the CUDA hot path (csrc/fastmath_tables.cuh) hold the correctly
rounded values they claim: 2^(j/64), rc_j = RN(1/(1 + (j + 1/2)/64)) and -log(rc_j) of the rounded rc_j.
Recomputed here with Python's decimal module at 50 digits (independent of the generator's 60)."""
import decimal
import math
import pathlib
import re

ROOT = pathlib.Path(__file__).resolve().parents[1]
HDR = ROOT / "paper_2510_23993_b200" / "csrc" / "fastmath_tables.cuh"


def _arrays():
    txt = HDR.read_text()
    exp2 = [float(v) for v in re.search(r"kExp2J\[64\] = \{([^}]*)\}", txt).group(1).split(",")]
    body = re.search(r"kLogTab\[64\] = \{(.*)\};", txt).group(1)
    pairs = [tuple(float(v) for v in m.split(",")) for m in re.findall(r"\{([^{}]*)\}", body)]
    return exp2, pairs


def test_tables_correctly_rounded():
    D = decimal.Decimal
    decimal.getcontext().prec = 50
    ln2 = D(2).ln()
    exp2, logtab = _arrays()
    assert len(exp2) == 64 and len(logtab) == 64
    for j in range(64):
        assert exp2[j] == float((ln2 * j / 64).exp()), j
        c = 1 + (D(j) + D(1) / 2) / 64
        rc, mlog = logtab[j]
        assert rc == float(1 / c), j
        assert mlog == float(-D(rc).ln()), j
        # z = m rc_j - 1 stays inside the polynomial's range |z| < 1/128 for m in [1 + j/64, 1 + (j+1)/64)
        for m in (1 + j / 64, 1 + (j + 1) / 64):
            assert abs(m * rc - 1) < 1 / 128 + 1e-15


def test_ln2_split():
    txt = HDR.read_text()
    hi = float(re.search(r"kLn2Hi = ([^;]*);", txt).group(1))
    lo = float(re.search(r"kLn2Lo = ([^;]*);", txt).group(1))
    decimal.getcontext().prec = 50
    ln2 = decimal.Decimal(2).ln()
    assert hi == math.log(2)
    assert abs((decimal.Decimal(hi) + decimal.Decimal(lo)) - ln2) < decimal.Decimal("1e-33")

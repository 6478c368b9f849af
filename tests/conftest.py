"""pytest configuration: the `gpu` marker and shared fixtures.

`-m "not gpu"` runs the oracle pins, host logic and the C-ABI symbol checks on CPU;
`-m gpu` runs the parity tests proper through the C-ABI on a B200.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer CPU pins (still part of the default suite)")


@pytest.fixture(scope="session")
def oracle_h2():
    from oracle import Oracle
    return Oracle("h2air_li2004")

"""paper_2510_23993_b200 — bulk-sparse stiff chemistry integration on B200 (sm_100a).

The product: libchem.so (hand-written CUDA for sm_100a behind the C ABI of include/chem.h) and a
thin torch binding.  See DESIGN.md.  This package never imports the oracle/ (test
infrastructure) and has no CPU fallback: calls fail loudly without the CUDA library.
"""
from .mechanism import MechTables, load as load_mechanism  # noqa: F401

__all__ = ["Chem", "Box", "load_mechanism", "MechTables"]


def __getattr__(name):
    # lazy: importing the package must not require torch/CUDA (the CPU test suite imports it)
    if name in ("Chem", "Box"):
        from . import api
        return getattr(api, name)
    raise AttributeError(name)

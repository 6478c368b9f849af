"""Build libchem.so in-tree: nvcc for sm_100a only (no other architectures, no JIT fallback).

    python -m paper_2510_23993_b200.build [--force]

Steps: regenerate the compile-time structure headers from mech/*.yaml (gen_structure), then
`nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared` of csrc/chem_api.cu.
"""
from __future__ import annotations

import os
import pathlib
import shutil
import subprocess
import sys

from . import gen_structure

PKG = pathlib.Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libchem.so"
INCLUDE = PKG.parent / "include"

NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found: libchem.so cannot be built")


def sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + sorted((CSRC / "mechs").glob("*.cuh")) + [
        INCLUDE / "chem.h"]


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(s.stat().st_mtime <= t for s in sources())


def build(force: bool = False, verbose: bool = False) -> pathlib.Path:
    gen_structure.generate()
    if not force and up_to_date():
        return LIB
    tmp = LIB.with_suffix(f".{os.getpid()}.tmp.so")
    cmd = [nvcc(), *NVCC_FLAGS, "-o", str(tmp), str(CSRC / "chem_api.cu")]
    r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    log = PKG / "build.log"
    log.write_text(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stderr[-5000:])
        raise RuntimeError(f"nvcc failed ({r.returncode}); see {log}")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    p = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(p)

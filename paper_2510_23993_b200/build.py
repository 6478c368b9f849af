"""Build libchem.so in-tree: nvcc for sm_100a only (no other architectures, no JIT fallback).

    python -m paper_2510_23993_b200.build [--force]

Steps: regenerate the compile-time structure headers from mech/*.yaml (gen_structure), compile every
csrc/*.cu translation unit (the C ABI in chem_api.cu, one launch_*.cu per integrator) with
`nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -c` in parallel, then link them with
`nvcc -shared`.
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
    "-Xcompiler", "-fPIC",
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


def _compile(src: pathlib.Path, obj: pathlib.Path):
    # CHEM_NVCC_EXTRA: extra flags for a kernel experiment (e.g. -DCHEM_...); the default build has none
    extra = os.environ.get("CHEM_NVCC_EXTRA", "").split()
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-c", "-o", str(obj), str(src)]
    r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    return src, cmd, r


def build(force: bool = False, verbose: bool = False) -> pathlib.Path:
    gen_structure.generate()
    if not force and up_to_date():
        return LIB
    import concurrent.futures as cf
    import tempfile
    tu = sorted(CSRC.glob("*.cu"))
    log_lines, failed = [], None
    with tempfile.TemporaryDirectory(prefix="chem_build_") as td:
        objs = [pathlib.Path(td) / (s.stem + ".o") for s in tu]
        with cf.ThreadPoolExecutor(max_workers=min(len(tu), os.cpu_count() or 4)) as ex:
            for src, cmd, r in ex.map(_compile, tu, objs):
                log_lines.append(" ".join(cmd) + "\n" + r.stdout + r.stderr)
                if r.returncode != 0 and failed is None:
                    failed = (src, r)
        if failed is None:
            tmp = LIB.with_suffix(f".{os.getpid()}.tmp.so")
            cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(tmp), *map(str, objs)]
            r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
            log_lines.append(" ".join(cmd) + "\n" + r.stdout + r.stderr)
            if r.returncode != 0:
                failed = ("link", r)
    log = PKG / "build.log"
    log.write_text("\n".join(log_lines))
    if failed is not None:
        sys.stderr.write(failed[1].stderr[-5000:])
        raise RuntimeError(f"nvcc failed on {failed[0]}; see {log}")
    if verbose:
        sys.stderr.write("\n".join(log_lines))
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    p = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(p)

"""Aggregate ncu warp-stall samples of a report by function region of chem_device.cuh/chem_kernels.cuh.

    python tools/ncu_regions.py gpurun_out/prof.ncu-rep
"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

ROOT = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))


def regions(fname):
    """(start_line, name) of each top-level function in a source file."""
    out = []
    for i, line in enumerate(open(f"{ROOT}/paper_2510_23993_b200/csrc/{fname}"), 1):
        m = re.match(r"__device__ __forceinline__ \S+ (\w+)\(|__global__ void .*? (k_\w+)\(|^\S.*\b(\w+)\($", line)
        m2 = re.search(r"(?:__forceinline__|__global__ void(?: __launch_bounds__\([^)]*\))?)\s+[\w:<>,*& ]*?\b(\w+)\(", line)
        if m2:
            out.append((i, m2.group(1)))
    return out


def main(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                         capture_output=True, text=True).stdout
    regs = {}
    f = None
    agg = Counter()
    tot = 0
    for r in csv.reader(io.StringIO(txt)):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            if f not in regs:
                try:
                    regs[f] = regions(f)
                except OSError:
                    regs[f] = []
            continue
        if r[0] in ("Line No", "-") or len(r) < 6:
            continue
        try:
            ln, s = int(r[0]), int(r[4])
        except ValueError:
            continue
        name = "?"
        for start, nm in regs.get(f, []):
            if start <= ln:
                name = nm
        agg[f"{f}:{name}"] += s
        tot += s
    for k, v in agg.most_common(30):
        print(f"{100 * v / max(tot, 1):6.1f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1])

"""Static SASS statistics of the kernels in a .so/.cubin: instruction count, FP64 ops, spills.

    python tools/sass_stats.py paper_2510_23993_b200/libchem.so [name-filter]
"""
import collections
import re
import subprocess
import sys


def main(path, filt=""):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    fn, stats = None, collections.OrderedDict()
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            fn = m.group(1)
            stats[fn] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if m and fn:
            stats[fn]["total"] += 1
            stats[fn][m.group(2)] += 1
    for fn, c in stats.items():
        if filt in fn:
            keys = ["DFMA", "DADD", "DMUL", "MUFU", "LDL", "STL", "LDS", "STS", "LDC", "BRA"]
            print(f"{fn[:90]:90s} total {c['total']:6d} " + " ".join(f"{k}={c[k]}" for k in keys))


if __name__ == "__main__":
    main(*sys.argv[1:])

"""Static SASS size of one kernel attributed to source functions (needs -lineinfo).

    python tools/sass_lines.py paper_2510_23993_b200/libchem.so <kernel-name-substring>
"""
import collections
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def regions(fname):
    out = []
    try:
        for i, line in enumerate(open(f"{ROOT}/paper_2510_23993_b200/csrc/{fname}"), 1):
            m = re.search(r"(?:__forceinline__|__global__ void(?: __launch_bounds__\([^)]*\))?)\s+[\w:<>,*& ]*?\b(\w+)\(",
                          line)
            if m:
                out.append((i, m.group(1)))
    except OSError:
        pass
    return out


def main(lib, name):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
    txt = ""
    for cubin in sorted(f for f in os.listdir(d) if f.endswith(".cubin")):   # one per translation unit
        txt += subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cubin)], capture_output=True, text=True).stdout
    lines = txt.splitlines()
    inside = False
    cur = None
    cnt = collections.Counter()
    total = 0
    for ln in lines:
        if ln.lstrip().startswith(".section") and ".text." in ln:
            inside = name in ln
            continue
        if not inside:
            continue
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        if re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
            total += 1
            cnt[cur] += 1
    regs = {}
    agg = collections.Counter()
    for key, c in cnt.items():
        if key is None:
            agg["?"] += c
            continue
        f, ln = key
        if f not in regs:
            regs[f] = regions(f)
        nm = "?"
        for s, n in regs[f]:
            if s <= ln:
                nm = n
        agg[f"{f}:{nm}"] += c
    print("total", total)
    for k, v in agg.most_common(20):
        print(f"{v:7d} {k}")


if __name__ == "__main__":
    main(*sys.argv[1:])

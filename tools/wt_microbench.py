"""w_t of SURVEY.md §8(d): the DADD + DMUL + 2*DFMA count of one libdevice exp / log on sm_100a.

Static count: compile tools/probes/fp64_probe.cu for sm_100a and count the FP64 instructions of the
k_exp / k_log kernels in the SASS (cuobjdump; no GPU needed).  The dynamic count per call (ncu
sm__sass_thread_inst_executed_op_{dadd,dmul,dfma}_pred_on.sum / elements) is added by
tools/fp64_probe.sh on the GPU box.  Writes profiles/wt_microbench.json.

    python tools/wt_microbench.py
"""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tools", "probes", "fp64_probe.cu")
BIN = os.path.join(ROOT, "tools", "probes", "fp64_probe")


def main():
    subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-o", BIN, SRC], check=True)
    sass = subprocess.run(["cuobjdump", "-sass", BIN], capture_output=True, text=True, check=True).stdout
    counts, cur = {}, None
    for line in sass.splitlines():
        m = re.search(r"Function : \S*(k_exp|k_log|dfma_peak)", line)
        if m:
            cur = m.group(1)
            counts[cur] = {"DADD": 0, "DMUL": 0, "DFMA": 0}
            continue
        if cur:
            for op in ("DADD", "DMUL", "DFMA"):
                if re.search(rf"\b{op}\b", line):
                    counts[cur][op] += 1
    out = {}
    for k, name in (("k_exp", "exp"), ("k_log", "log")):
        c = counts[k]
        out[name] = dict(c, w_t=c["DADD"] + c["DMUL"] + 2 * c["DFMA"])
    doc = {"what": "DADD + DMUL + 2*DFMA of one libdevice exp/log call, sm_100a SASS (SURVEY §8(d) w_t)",
           "static": out, "source": "tools/probes/fp64_probe.cu, nvcc 12.9 -O3 sm_100a"}
    path = os.path.join(ROOT, "profiles", "wt_microbench.json")
    if os.path.exists(path):
        old = json.load(open(path))
        if "dynamic" in old:
            doc["dynamic"] = old["dynamic"]
    json.dump(doc, open(path, "w"), indent=1)
    print(json.dumps(doc))
    return 0


if __name__ == "__main__":
    sys.exit(main())

"""Top source lines of an ncu report by warp-stall samples (ncu --page source, cuda+sass view).

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys


def main(rep, n=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                         capture_output=True, text=True).stdout
    f = None
    rows = []
    hdr = None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and r[0] != "-" and len(r) > 6:
            try:
                samples = int(r[4])
                execd = int(r[7])
            except ValueError:
                continue
            rows.append((samples, execd, f, r[0], r[1][:90], r[13] if len(r) > 13 else ""))
    tot = sum(x[0] for x in rows) or 1
    for s, e, f, ln, src, sp in sorted(rows, reverse=True)[: int(n)]:
        print(f"{100 * s / tot:5.1f}% {e:11d} {f}:{ln:5s} {src:90s} {sp[:40]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
